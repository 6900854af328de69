// Step Rehash similarity: the K x K Gram matrix of the K cached probe tensors in ONE pass
// over HBM (cosine_similarity, kernels.py:375-390; similarity map).
//
// G = P P^T with P the K x n matrix of probes (n = 73.7M elements at SVD-XT shape).  The
// contraction is HBM-bound (K = 25: 3.7 GB of bf16 probes per map), so the kernel is built to
// read every probe element exactly once: each warp walks a contiguous element range 16 at a
// time and feeds the same registers to both operands of bf16 mma.sync m16n8k16 (A = rows of
// P, B = the same rows as P^T columns).  Products of bf16 values are exact in fp32; the fp32
// MMA accumulators are flushed into fp64 every 16 k-steps (256 elements), warps are combined
// in fixed order through shared memory and blocks in fixed order by the finalize kernel --
// bit-reproducible, no atomics.
//
// K <= 32 runs as one 32 x 32 job; larger K as jobs over pairs of 32-probe blocks (gridDim.y).
// A row >= K reads as zero.  The n % 16 tail is added in fp64 by block 0.
#include "common.cuh"

namespace sf {
namespace gram {

constexpr int WARPS = 8, THREADS = WARPS * 32;
constexpr int KSTEP = 16, UNROLL = 4, FLUSH = 16;   // flush every FLUSH k-steps

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ uint32_t ld_u32(const bf16* p) {
  uint32_t v;
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// job (bi, bj), bi <= bj, of nb 32-probe blocks
__device__ __forceinline__ void job_of(int y, int nb, int& bi, int& bj) {
  bi = 0;
  while (y >= nb - bi) {
    y -= nb - bi;
    ++bi;
  }
  bj = bi + y;
}

// part[(blockIdx.y * gridDim.x + blockIdx.x) * 1024 + i * 32 + j]: this block's 32x32 partial
__global__ void __launch_bounds__(THREADS) gram_mma_kernel(const bf16* const* __restrict__ probes, int K, int64_t n,
                                                            double* __restrict__ part) {
  griddep_wait();
  griddep_trigger();
  const int nb = (K + 31) / 32;
  int bi, bj;
  job_of(blockIdx.y, nb, bi, bj);
  const bool diag = bi == bj;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c0 = (lane & 3) * 2;
  // the 4 probe rows this thread loads for the A side (block bi) and the B side (block bj)
  const bf16* pa[4];
  const bf16* pb[4];
  bool va[4], vb[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ia = bi * 32 + g + 8 * r, ib = bj * 32 + g + 8 * r;
    va[r] = ia < K;
    vb[r] = ib < K;
    pa[r] = probes[va[r] ? ia : 0] + c0;
    pb[r] = probes[vb[r] ? ib : 0] + c0;
  }
  const int64_t nsteps = n / KSTEP;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  const int64_t per = (nsteps + nw - 1) / nw;
  const int64_t s0 = gw * per, s1 = s0 + per < nsteps ? s0 + per : nsteps;

  double acc[2][4][4];
  float c[2][4][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[m][t][e] = 0.0;
        c[m][t][e] = 0.f;
      }
  int since = 0;
  for (int64_t s = s0; s < s1; s += UNROLL) {
    const int nk = (int)(s1 - s < UNROLL ? s1 - s : UNROLL);
    uint32_t LA[UNROLL][4][2], LB[UNROLL][4][2];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (u < nk) {
        const int64_t e0 = (s + u) * KSTEP;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          LA[u][r][0] = va[r] ? ld_u32(pa[r] + e0) : 0u;
          LA[u][r][1] = va[r] ? ld_u32(pa[r] + e0 + 8) : 0u;
          if (!diag) {
            LB[u][r][0] = vb[r] ? ld_u32(pb[r] + e0) : 0u;
            LB[u][r][1] = vb[r] ? ld_u32(pb[r] + e0 + 8) : 0u;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (u < nk) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const uint32_t a[4] = {LA[u][2 * m][0], LA[u][2 * m + 1][0], LA[u][2 * m][1], LA[u][2 * m + 1][1]};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const uint32_t b[2] = {diag ? LA[u][t][0] : LB[u][t][0], diag ? LA[u][t][1] : LB[u][t][1]};
            mma16816(c[m][t], a, b);
          }
        }
      }
    }
    since += nk;
    if (since >= FLUSH) {
      since = 0;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[m][t][e] += (double)c[m][t][e];
            c[m][t][e] = 0.f;
          }
    }
  }
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[m][t][e] += (double)c[m][t][e];

  // fixed-order combine of the 8 warps into one 32x32 tile (warp 0 first, then 1, ...)
  __shared__ double tile[32 * 32];
  for (int w = 0; w < WARPS; ++w) {
    if (warp == w) {
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int idx = (m * 16 + g + (e >= 2 ? 8 : 0)) * 32 + t * 8 + c0 + (e & 1);
            tile[idx] = (w == 0 ? 0.0 : tile[idx]) + acc[m][t][e];
          }
    }
    __syncthreads();
  }
  double* out = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 1024;
  for (int i = threadIdx.x; i < 1024; i += THREADS) out[i] = tile[i];
  // the n % 16 tail elements, block 0 of every job
  if (blockIdx.x == 0 && nsteps * KSTEP < n) {
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += THREADS) {
      const int ri = bi * 32 + i / 32, rj = bj * 32 + i % 32;
      if (ri < K && rj < K) {
        double v = 0.0;
        for (int64_t e = nsteps * KSTEP; e < n; ++e)
          v += (double)__bfloat162float(probes[ri][e]) * (double)__bfloat162float(probes[rj][e]);
        out[i] += v;
      }
    }
  }
}

// out[i*K + j] = sum over blocks (fixed order) of the job's partials, mirrored
__global__ void gram_combine_kernel(const double* __restrict__ part, int K, int nblk, double* __restrict__ out) {
  griddep_wait();
  griddep_trigger();
  const int nb = (K + 31) / 32;
  int bi, bj;
  job_of(blockIdx.x, nb, bi, bj);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    const int ri = bi * 32 + i / 32, rj = bj * 32 + i % 32;
    if (ri >= K || rj >= K) continue;
    double v = 0.0;
    const double* p = part + (int64_t)blockIdx.x * nblk * 1024 + i;
    for (int b = 0; b < nblk; ++b) v += p[(int64_t)b * 1024];
    if (bi != bj || ri <= rj) {
      out[(int64_t)ri * K + rj] = v;
      out[(int64_t)rj * K + ri] = v;
    }
  }
}

inline int blocks_per_job() { return num_sms(); }   // one 8-warp block per SM (232 registers)

}  // namespace gram
}  // namespace sf

using namespace sf;

extern "C" {

int64_t sf_gram_workspace(int32_t K, int64_t n) {
  (void)n;
  const int64_t nb = (K + 31) / 32, jobs = nb * (nb + 1) / 2;
  return jobs * gram::blocks_per_job() * 1024 * (int64_t)sizeof(double);
}

sf_status sf_gram_bf16(const void* const* probes, int32_t K, int64_t n, void* work, double* out, void* stream) {
  SF_CHECK_ARG(K >= 1 && n >= 1 && probes && work && out, SF_ERR_SHAPE, "bad extents");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (K + 31) / 32, jobs = nb * (nb + 1) / 2, nblk = gram::blocks_per_job();
  launch_k(gram::gram_mma_kernel, dim3(nblk, jobs), dim3(gram::THREADS), 0, st, (const bf16* const*)probes, (int)K, n,
           (double*)work);
  launch_k(gram::gram_combine_kernel, dim3(jobs), dim3(256), 0, st, (const double*)work, (int)K, nblk, out);
  return launch_status("sf_gram_bf16");
}

}  // extern "C"
