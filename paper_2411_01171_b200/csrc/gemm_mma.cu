// Generic implicit GEMM on the legacy warp-level tensor path (mma.sync
// m16n8k16 bf16 -> fp32).  Handles every shape of the sliceflow contractions:
// any channel count that is a multiple of 8, 3x3 / 3-tap-temporal implicit
// im2col, K-major or MN-major weights, two-level row views, batching.
//
// This is the portable fallback and the correctness baseline; the tcgen05/TMA
// kernel in gemm_tc.cu takes every shape whose channel counts are multiples of
// 64 (all SD-width configurations).
#include "common.cuh"

namespace sf {
namespace mma {

constexpr int BM = 128, BN = 128, BK = 32, THREADS = 256;
constexpr int APAD = 8;                 // row pad (elements) against ldmatrix bank conflicts
constexpr int AS = BK + APAD;           // A/B(K-major) smem row stride
constexpr int BSN = BN + 8;             // B (MN-major) smem row stride

struct Smem {
  bf16 a[2][BM][AS];
  union {
    bf16 bk[2][BN][AS];   // K-major weights  [n][k]
    bf16 bn[2][BK][BSN];  // MN-major weights [k][n]
  } b;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void ldsm_x4(unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3, const void* p) {
  unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3, const void* p) {
  unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(s));
}
__device__ __forceinline__ void mma16816(float* c, const unsigned* a, unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Address of A element (m, k0..k0+7) for the implicit-GEMM modes; nullptr = zero.
__device__ __forceinline__ const bf16* a_addr(const sf_gemm_args& p, const bf16* base, int64_t m, int k0, int K) {
  const int64_t M = (int64_t)p.n_outer * p.n_inner;
  if (m >= M || k0 >= K) return nullptr;
  int64_t o = m / p.n_inner;
  int64_t i = m - o * p.n_inner;
  int tap = k0 / p.cin, c = k0 - tap * p.cin;
  if (p.mode == SF_GEMM_CONV3X3) {
    int y = (int)(i / p.W) + tap / 3 - 1, x = (int)(i % p.W) + tap % 3 - 1;
    if (y < 0 || y >= p.H || x < 0 || x >= p.W) return nullptr;
    i = (int64_t)y * p.W + x;
  } else if (p.mode == SF_GEMM_TCONV3) {
    int t = (int)(o % p.T) + tap - 1;
    if (t < 0 || t >= p.T) return nullptr;
    o += tap - 1;
  }
  return base + (o * p.a.ostride + i) * p.a.ld + c;
}

template <bool WK>
__global__ void __launch_bounds__(THREADS) gemm_kernel(const __grid_constant__ sf_gemm_args p) {
  griddep_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, 64 x 32 each
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const int taps = p.mode == SF_GEMM_PLAIN ? 1 : (p.mode == SF_GEMM_CONV3X3 ? 9 : 3);
  const int K = taps * p.cin;
  const bf16* A = reinterpret_cast<const bf16*>(p.a.ptr) + (int64_t)z * p.a_bstride;
  const bf16* Wt = reinterpret_cast<const bf16*>(p.w) + (int64_t)z * p.w_bstride;

  auto load_stage = [&](int st, int kt) {
    const int kb = kt * BK;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      int v = tid + r * THREADS;          // 512 vectors: 128 rows x 4
      int row = v >> 2, kv = (v & 3) * 8;
      const bf16* src = a_addr(p, A, m0 + row, kb + kv, K);
      cp_async16(&sm.a[st][row][kv], src ? src : A, src != nullptr);
    }
    if (WK) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        int v = tid + r * THREADS;
        int n = v >> 2, kv = (v & 3) * 8;
        bool ok = (n0 + n) < p.N && (kb + kv) < K;
        const bf16* src = Wt + (int64_t)(n0 + n) * p.w_ld + kb + kv;
        cp_async16(&sm.b.bk[st][n][kv], ok ? src : Wt, ok);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        int v = tid + r * THREADS;          // 32 k-rows x 16 vectors
        int k = v >> 4, nv = (v & 15) * 8;
        bool ok = (kb + k) < K && (n0 + nv) < p.N;
        const bf16* src = Wt + (int64_t)(kb + k) * p.w_ld + n0 + nv;
        cp_async16(&sm.b.bn[st][k][nv], ok ? src : Wt, ok);
      }
    }
  };

  float acc[4][4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.f;

  const int KT = (K + BK - 1) / BK;
  load_stage(0, 0);
  cp_commit();
  for (int kt = 0; kt < KT; ++kt) {
    const int st = kt & 1;
    if (kt + 1 < KT) load_stage(st ^ 1, kt + 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 16) {
      unsigned af[4][4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        int r = wm * 64 + mi * 16 + (lane & 15);
        int c = kk + (lane >> 4) * 8;
        ldsm_x4(af[mi][0], af[mi][1], af[mi][2], af[mi][3], &sm.a[st][r][c]);
      }
      unsigned bfr[4][2];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        unsigned r0, r1, r2, r3;
        if (WK) {
          // rows n (16 of them), cols k: matrices (n0-7,k0-7),(n0-7,k8-15),(n8-15,k0-7),(n8-15,k8-15)
          int n = wn * 32 + nj * 16 + (lane & 7) + ((lane >> 4) << 3);
          int c = kk + ((lane >> 3) & 1) * 8;
          ldsm_x4(r0, r1, r2, r3, &sm.b.bk[st][n][c]);
        } else {
          // smem [k][n]; transpose loads: matrices (k0-7,n..),(k8-15,n..),(k0-7,n+8..),(k8-15,n+8..)
          int k = kk + (lane & 7) + ((lane >> 3) & 1) * 8;
          int n = wn * 32 + nj * 16 + (lane >> 4) * 8;
          ldsm_x4_t(r0, r1, r2, r3, &sm.b.bn[st][k][n]);
        }
        bfr[nj * 2 + 0][0] = r0;
        bfr[nj * 2 + 0][1] = r1;
        bfr[nj * 2 + 1][0] = r2;
        bfr[nj * 2 + 1][1] = r3;
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma16816(acc[mi][ni], af[mi], bfr[ni][0], bfr[ni][1]);
    }
    __syncthreads();
  }

  // epilogue
  const int64_t M = (int64_t)p.n_outer * p.n_inner;
  const bf16* R = reinterpret_cast<const bf16*>(p.res.ptr);
  unsigned char* Ob = reinterpret_cast<unsigned char*>(p.out.ptr) +
                      (int64_t)z * p.out_bstride * (p.out_fp32 ? 4 : 2);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t m = m0 + wm * 64 + mi * 16 + (lane >> 2) + h * 8;
      if (m >= M) continue;
      int64_t o = m / p.n_inner, i = m - o * p.n_inner;
      int64_t orow = (o * p.out.ostride + i) * p.out.ld;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        int n = n0 + wn * 32 + ni * 8 + (lane & 3) * 2;
        if (n >= p.N) continue;
        float v0 = acc[mi][ni][h * 2 + 0], v1 = acc[mi][ni][h * 2 + 1];
        bool two = n + 1 < p.N;
        if (p.rowstats) {   // folded LayerNorm: rstd * (acc - mean * colsum)
          const float2 s = reinterpret_cast<const float2*>(p.rowstats)[m];
          v0 = fmaf(s.x, v0, s.y * p.colvec[n]);
          if (two) v1 = fmaf(s.x, v1, s.y * p.colvec[n + 1]);
        }
        v0 *= p.alpha;
        v1 *= p.alpha;
        if (p.bias) {
          v0 += p.bias[n];
          if (two) v1 += p.bias[n + 1];
        }
        if (p.rowbias) {
          const float* rb = p.rowbias + o * p.rowbias_stride;
          v0 += rb[n];
          if (two) v1 += rb[n + 1];
        }
        if (p.act == SF_ACT_SILU) {
          v0 = silu_f(v0);
          v1 = silu_f(v1);
        }
        if (R) {
          const bf16* rr = R + (int64_t)z * p.res_bstride + (o * p.res.ostride + i) * p.res.ld + n;
          v0 += __bfloat162float(rr[0]);
          if (two) v1 += __bfloat162float(rr[1]);
        }
        if (p.out_fp32) {
          float* dst = reinterpret_cast<float*>(Ob) + orow + n;
          if (two && ((orow + n) & 1) == 0) {
            *reinterpret_cast<float2*>(dst) = make_float2(v0, v1);
          } else {
            dst[0] = v0;
            if (two) dst[1] = v1;
          }
        } else {
          bf16* dst = reinterpret_cast<bf16*>(Ob) + orow + n;
          if (two && ((orow + n) & 1) == 0) {
            *reinterpret_cast<bf162*>(dst) = __floats2bfloat162_rn(v0, v1);
          } else {
            dst[0] = __float2bfloat16(v0);
            if (two) dst[1] = __float2bfloat16(v1);
          }
        }
      }
    }
  }
}

}  // namespace mma

sf_status gemm_mma_launch(const sf_gemm_args& p, cudaStream_t st) {
  const int64_t M = (int64_t)p.n_outer * p.n_inner;
  dim3 grid((unsigned)((M + mma::BM - 1) / mma::BM), (unsigned)((p.N + mma::BN - 1) / mma::BN),
            (unsigned)p.batch);
  size_t smem = sizeof(mma::Smem);
  if (p.w_kmajor) {
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(mma::gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      init = true;
    }
    launch_k(mma::gemm_kernel<true>, dim3(grid), dim3(mma::THREADS), smem, st, p);
  } else {
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(mma::gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      init = true;
    }
    launch_k(mma::gemm_kernel<false>, dim3(grid), dim3(mma::THREADS), smem, st, p);
  }
  return launch_status("sf_gemm(mma.sync)");
}

}  // namespace sf
