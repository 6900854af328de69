// Fused single-head spatial attention, version 2 (kernels.py:269-300):
//   O = softmax(Q K^T * scale) V per frame, head_dim D = C <= 320.
//
// Built around the shared-memory port, which the v1 profile showed to be the
// limit (SS-mode MMAs re-read Q for every key block, P was written and read
// twice through smem, and TMA writes K/V into the same port):
//   * 128-key blocks: Q is re-read once per 128 keys instead of per 64;
//   * P lives in TMEM and is the A operand of P.V (tcgen05.mma A-from-TMEM):
//     no P smem traffic at all;
//   * K_j / V^T_j stream through a 7-slot ring of 20 KB items (one 64-wide d
//     chunk of K_j, or one [D/2 x 64 keys] quarter of V^T_j) so loads run
//     several items ahead of the tensor core.
// TMEM: O [0,D) fp32 | S [320,448) fp32 (one 128-key block) | P [448,512) bf16x2.
// Warps: 0 TMA, 1 MMA issuer (+TMEM alloc), 2..5 softmax + epilogue (one row each).
#include "common.cuh"

#include <cuda.h>
#include <mutex>

namespace sf {
namespace fa2 {

constexpr int BQ = 128, BKV = 128, THREADS = 192;
constexpr int NSLOT = 7, SLOT_BYTES = 20480;
constexpr int O_COL = 0, S_COL = 320, P_COL = 448;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma3(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// D[tmem] (+)= A[smem] B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// D[tmem] (+)= A[tmem] B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define SF_R32(r) \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
      "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), \
      "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), \
      "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define SF_W32(r) \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), \
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), \
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), \
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])

__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : SF_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      SF_W32(r));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct Params {
  int HW, frames, n_kv;
  float scale_log2;
  sf_view_t out;
};

template <int D>
struct Layout {
  static constexpr int NCH = D / 64;
  static constexpr int Q_BYTES = NCH * BQ * 128;
  static constexpr int K_ITEM = BKV * 128;        // [128 keys x 64 d]
  static constexpr int V_ITEM = (D / 2) * 128;    // [D/2 d x 64 keys]
  static constexpr int TOTAL = 1024 + Q_BYTES + NSLOT * SLOT_BYTES + 256;
  static_assert(K_ITEM <= SLOT_BYTES && V_ITEM <= SLOT_BYTES, "ring slot too small");
  static_assert(D % 64 == 0 && D <= 320 && (D / 2) % 16 == 0, "head dim");
};

// ring item sequence shared by the TMA warp and the MMA warp:
//   K_0[0..NCH), then per block j: K_{j+1}[0..NCH) (if any), V_j[(kc,h) for kc<2, h<2]
template <int D>
__global__ void __launch_bounds__(THREADS, 1)
    flash2_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap mQ,
                  const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV) {
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;
  uint8_t* sRing = sQ + L::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRing + NSLOT * SLOT_BYTES);
  uint64_t* q_full = bars;
  uint64_t* r_full = bars + 1;          // [NSLOT]
  uint64_t* r_empty = r_full + NSLOT;   // [NSLOT]
  uint64_t* s_full = r_empty + NSLOT;
  uint64_t* s_empty = s_full + 1;
  uint64_t* p_full = s_empty + 1;
  uint64_t* o_done = p_full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * BQ, f = blockIdx.y;
  const int nkv = p.n_kv;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 4);
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  // prologue (barriers, TMEM) done without touching global data: now wait for the
  // producing kernel (PDL) and let the next one be scheduled
  griddep_wait();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, L::Q_BYTES);
      for (int c = 0; c < L::NCH; ++c) tma3(&mQ, q_full, sQ + c * BQ * 128, c * 64, q0, f);
      int slot = 0;
      uint32_t ph = 0;
      auto next = [&]() {
        if (++slot == NSLOT) {
          slot = 0;
          ph ^= 1;
        }
      };
      auto load_k = [&](int j) {
        for (int c = 0; c < L::NCH; ++c) {
          mbar_wait(&r_empty[slot], ph ^ 1);
          mbar_expect_tx(&r_full[slot], L::K_ITEM);
          tma3(&mK, &r_full[slot], sRing + slot * SLOT_BYTES, c * 64, j * BKV, f);
          next();
        }
      };
      load_k(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) load_k(j + 1);
        for (int kc = 0; kc < 2; ++kc)
          for (int h = 0; h < 2; ++h) {
            mbar_wait(&r_empty[slot], ph ^ 1);
            mbar_expect_tx(&r_full[slot], L::V_ITEM);
            tma3(&mV, &r_full[slot], sRing + slot * SLOT_BYTES, j * BKV + kc * 64, h * (D / 2), f);
            next();
          }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc(BKV), idO = idesc(D / 2);
      mbar_wait(q_full, 0);
      fence_after();
      const uint64_t qd = sdesc(smem_u32(sQ));
      int slot = 0;
      uint32_t ph = 0;
      auto next = [&]() {
        if (++slot == NSLOT) {
          slot = 0;
          ph ^= 1;
        }
      };
      auto issue_S = [&](int j) {
        mbar_wait(s_empty, (j & 1) ^ 1);  // softmax of block j-1 has read S out of TMEM
        fence_after();
#pragma unroll 1
        for (int c = 0; c < L::NCH; ++c) {
          mbar_wait(&r_full[slot], ph);
          fence_after();
          const uint64_t kd = sdesc(smem_u32(sRing + slot * SLOT_BYTES));
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ss(tmem + S_COL, qd + (uint64_t)((c * BQ * 128 + k * 32) >> 4), kd + (uint64_t)(2 * k), idS,
                   (c | k) != 0);
          commit(&r_empty[slot]);
          next();
        }
        commit(s_full);
      };
      auto issue_PV = [&](int j) {
        mbar_wait(p_full, j & 1);
        fence_after();
#pragma unroll 1
        for (int kc = 0; kc < 2; ++kc) {
          const int s0 = slot;
          mbar_wait(&r_full[slot], ph);
          next();
          const int s1 = slot;
          mbar_wait(&r_full[slot], ph);
          next();
          fence_after();
          const uint64_t v0 = sdesc(smem_u32(sRing + s0 * SLOT_BYTES));
          const uint64_t v1 = sdesc(smem_u32(sRing + s1 * SLOT_BYTES));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t pa = tmem + P_COL + (uint32_t)((kc * 64 + k * 16) / 2);
            mma_ts(tmem + O_COL, pa, v0 + (uint64_t)(2 * k), idO, (j | kc | k) != 0);
            mma_ts(tmem + O_COL + D / 2, pa, v1 + (uint64_t)(2 * k), idO, (j | kc | k) != 0);
          }
          commit(&r_empty[s0]);
          commit(&r_empty[s1]);
        }
        commit(o_done);
      };
      issue_S(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_S(j + 1);
        issue_PV(j);
      }
    }
  } else {
    // ================= softmax + epilogue: one query row per thread =================
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float c = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      fence_after();
      uint32_t r[BKV];
#pragma unroll
      for (int k = 0; k < BKV / 32; ++k) tld32(tmem + lane_off + S_COL + 32 * k, r + 32 * k);
      tld_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      const int kbase = j * BKV;
      if (kbase + BKV > p.HW) {  // ragged last block: mask keys beyond the sequence
#pragma unroll
        for (int e = 0; e < BKV; ++e)
          if (kbase + e >= p.HW) r[e] = __float_as_uint(-INFINITY);
      }
      float mraw = -INFINITY;  // max of raw scores; scale c > 0 commutes with max
#pragma unroll
      for (int e = 0; e < BKV; e += 2) mraw = fmaxf(mraw, fmaxf(__uint_as_float(r[e]), __uint_as_float(r[e + 1])));
      const float mb = mraw * c;
      bool need = false;
      float corr = 1.f;
      if (j == 0) {
        m_run = mb;
      } else if (mb > m_run + 8.f) {  // lazy rescale (factor <= 2^8 otherwise)
        need = true;
        corr = ex2(m_run - mb);
        m_run = mb;
      }
      float ls0 = 0.f, ls1 = 0.f;
      uint32_t pk[BKV / 2];
#pragma unroll
      for (int e = 0; e < BKV / 2; ++e) {
        const float a = ex2(fmaf(__uint_as_float(r[2 * e]), c, -m_run));
        const float b = ex2(fmaf(__uint_as_float(r[2 * e + 1]), c, -m_run));
        ls0 += a;
        ls1 += b;
        bf162 h = __floats2bfloat162_rn(a, b);
        pk[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      const float ls = ls0 + ls1;
      // P.V of block j-1 must be done: P is overwritten below and O may be rescaled
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        fence_after();
      }
      if (__any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          tld32(tmem + lane_off + O_COL + cc, o);
          tld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tst32(tmem + lane_off + O_COL + cc, o);
        }
      }
      tst32(tmem + lane_off + P_COL, pk);
      tst32(tmem + lane_off + P_COL + 32, pk + 32);
      tst_wait();
      l_run = l_run * corr + ls;
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(o_done, (nkv - 1) & 1);
    fence_after();
    const float inv = 1.f / l_run;
    const int qrow = q0 + row;
    const bool valid = qrow < p.HW;
    bf16* dst = reinterpret_cast<bf16*>(p.out.ptr) + ((int64_t)f * p.out.ostride + qrow) * p.out.ld;
#pragma unroll 1
    for (int cc = 0; cc < D; cc += 32) {
      uint32_t o[32];
      tld32(tmem + lane_off + O_COL + cc, o);
      tld_wait();
      if (valid) {
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(o[e]) * inv;
#pragma unroll
        for (int e = 0; e < 4; ++e) reinterpret_cast<bf16x8*>(dst + cc)[e] = pack8(v + 8 * e);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}
static bool enc3(CUtensorMap* m, const void* g, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                 uint32_t b0, uint32_t b1) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2}, str[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1}, es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(g), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
static sf_status launch(const Params& p, const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                        cudaStream_t st) {
  constexpr int smem = Layout<D>::TOTAL;
  static_assert(smem <= 232448, "shared memory budget");
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(flash2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  dim3 grid((p.HW + BQ - 1) / BQ, p.frames);
  launch_k(flash2_kernel<D>, dim3(grid), dim3(THREADS), smem, st, p, q, k, v);
  return launch_status("sf_spatial_attention_core(v2)");
}

}  // namespace fa2

sf_status flash2_launch(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int frames, int HW, int C,
                        float scale, cudaStream_t st) {
  fa2::Params p{};
  p.HW = HW;
  p.frames = frames;
  p.n_kv = (HW + fa2::BKV - 1) / fa2::BKV;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  const uint64_t es = 2;
  const uint64_t qst = (uint64_t)(q.ostride ? q.ostride : HW) * q.ld * es;
  CUtensorMap mq, mk, mv;
  SF_CHECK_ARG(fa2::enc3(&mq, q.ptr, C, HW, frames, q.ld * es, qst, 64, fa2::BQ), SF_ERR_CUDA, "tensor map Q");
  SF_CHECK_ARG(fa2::enc3(&mk, k.ptr, C, HW, frames, k.ld * es, qst, 64, fa2::BKV), SF_ERR_CUDA, "tensor map K");
  SF_CHECK_ARG(fa2::enc3(&mv, vt, HW, C, frames, (uint64_t)HW * es, (uint64_t)C * HW * es, 64, C / 2), SF_ERR_CUDA,
               "tensor map V");
  switch (C) {
    case 320: return fa2::launch<320>(p, mq, mk, mv, st);
    case 256: return fa2::launch<256>(p, mq, mk, mv, st);
    case 192: return fa2::launch<192>(p, mq, mk, mv, st);
    default: return fa2::launch<128>(p, mq, mk, mv, st);
  }
}

}  // namespace sf
