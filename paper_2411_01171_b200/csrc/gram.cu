// Step Rehash similarity: the K x K Gram matrix of the K cached probe tensors in ONE pass
// over HBM (cosine_similarity, kernels.py:375-390; similarity map).
//
// G = P P^T with P the K x n matrix of probes (n = 73.7M elements at SVD-XT shape).  The
// contraction is HBM-bound (K = 25: 3.7 GB of bf16 probes per map), so the kernel is built to
// read every probe element exactly once: each warp walks a contiguous element range 32 at a
// time (16-byte loads, 4 lanes x 16 B per row) and feeds the same registers to both operands of
// bf16 mma.sync m16n8k16 (A = rows of P, B = the same rows as P^T columns).  Products of bf16
// values are exact; the MMA's fp32 accumulators are flushed into thread-private fp64 shared-
// memory accumulators every 16 k-steps (256 elements), warps are combined
// in fixed order through shared memory and blocks in fixed order by the combine kernel --
// bit-reproducible, no atomics.
//
// K <= 32 runs as one 32 x 32 job; larger K as one launch per pair of 32-probe blocks.
// Every probe must be 16-byte aligned (n % 8 == 0 for probes packed back to back).
// A row >= K reads as zero.  The n % 16 tail is added in fp64 by block 0.
#include "common.cuh"

namespace sf {
namespace gram {

constexpr int WARPS = 8, THREADS = WARPS * 32;
constexpr int CHUNK = 32;        // elements per row per warp load (4 lanes x 16 B) = 2 mma k-steps
constexpr int UNROLL = 4;        // 16-byte loads per probe row in flight per thread
constexpr int FLUSH = 2;         // loop iterations (2*UNROLL k-steps each) between fp64 flushes

__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ld16(const bf16* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
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

// One k-step (half h of a 16-byte load): the Gram is invariant under any permutation of the
// element index applied to every row alike, so lane (g, q) feeds its 8 loaded elements
// e0..e7 (offset 8q of a 32-element chunk) as k-slots {2q, 2q+1} <- e[4h], e[4h+1] and
// {2q+8, 2q+9} <- e[4h+2], e[4h+3]: each chunk is two complete m16n8k16 k-steps.
template <bool DIAG>
__device__ __forceinline__ void kstep(float (&c)[2][4][4], const uint4* LA, const uint4* LB, int h) {
  uint32_t a0[4], a1[4], b0[4], b1[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    a0[r] = h ? LA[r].z : LA[r].x;
    a1[r] = h ? LA[r].w : LA[r].y;
    b0[r] = DIAG ? a0[r] : (h ? LB[r].z : LB[r].x);
    b1[r] = DIAG ? a1[r] : (h ? LB[r].w : LB[r].y);
  }
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < 4; ++t) mma16816(c[m][t], a0[2 * m], a0[2 * m + 1], a1[2 * m], a1[2 * m + 1], b0[t], b1[t]);
}

// part[(job * gridDim.x + blockIdx.x) * 1024 + i * 32 + j]: this block's 32x32 partial of job (bi, bj)
template <bool DIAG>
__global__ void __launch_bounds__(THREADS, 2) gram_mma_kernel(const bf16* const* __restrict__ probes, int K, int64_t n,
                                                               int job, double* __restrict__ part) {
  griddep_wait();
  griddep_trigger();
  extern __shared__ double sacc[];   // [WARPS][32 entries][32 lanes]: thread-private fp64 accumulators
  const int nb = (K + 31) / 32;
  int bi, bj;
  job_of(job, nb, bi, bj);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  double* my = sacc + warp * 1024 + lane;
#pragma unroll
  for (int i = 0; i < 32; ++i) my[i * 32] = 0.0;
  const bf16* pa[4];
  const bf16* pb[4];
  bool va[4], vb[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int ia = bi * 32 + g + 8 * r, ib = bj * 32 + g + 8 * r;
    va[r] = ia < K;
    vb[r] = ib < K;
    pa[r] = probes[va[r] ? ia : 0] + 8 * q;
    pb[r] = probes[vb[r] ? ib : 0] + 8 * q;
  }
  const int64_t nchunks = n / CHUNK;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  const int64_t per = (nchunks + nw - 1) / nw;
  const int64_t s0 = gw * per, s1 = s0 + per < nchunks ? s0 + per : nchunks;
  float c[2][4][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) c[m][t][e] = 0.f;
  const uint4 zero = make_uint4(0, 0, 0, 0);
  int it = 0;
  for (int64_t s = s0; s < s1; s += UNROLL) {
    uint4 LA[UNROLL][4], LB[UNROLL][4];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const bool in = s + u < s1;
      const int64_t e0 = (s + u) * CHUNK;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        LA[u][r] = in && va[r] ? ld16(pa[r] + e0) : zero;
        if (!DIAG) LB[u][r] = in && vb[r] ? ld16(pb[r] + e0) : zero;
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      kstep<DIAG>(c, LA[u], DIAG ? LA[u] : LB[u], 0);
      kstep<DIAG>(c, LA[u], DIAG ? LA[u] : LB[u], 1);
    }
    if (++it == FLUSH || s + UNROLL >= s1) {
      it = 0;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            my[((m * 4 + t) * 4 + e) * 32] += (double)c[m][t][e];
            c[m][t][e] = 0.f;
          }
    }
  }
  __syncthreads();
  // fixed-order combine: entry (m,t,e) of lane L of warp w is Gram element (row, col) below
  double* out = part + ((int64_t)job * gridDim.x + blockIdx.x) * 1024;
  for (int idx = threadIdx.x; idx < 1024; idx += THREADS) {
    const int L = idx & 31, slot = idx >> 5;          // slot = (m*4 + t)*4 + e
    const int m = slot >> 4, t = (slot >> 2) & 3, e = slot & 3;
    const int row = m * 16 + (L >> 2) + (e >= 2 ? 8 : 0), col = t * 8 + (L & 3) * 2 + (e & 1);
    double v = 0.0;
    for (int w = 0; w < WARPS; ++w) v += sacc[w * 1024 + slot * 32 + L];
    out[row * 32 + col] = v;
  }
  // the n % 32 tail elements, block 0 of every job
  if (blockIdx.x == 0 && nchunks * CHUNK < n) {
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += THREADS) {
      const int ri = bi * 32 + i / 32, rj = bj * 32 + i % 32;
      if (ri < K && rj < K) {
        double v = 0.0;
        for (int64_t e = nchunks * CHUNK; e < n; ++e)
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

inline int blocks_per_job() { return num_sms() * 2; }   // two 8-warp blocks per SM
constexpr int SMEM = WARPS * 1024 * (int)sizeof(double);

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
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(gram::gram_mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, gram::SMEM);
    cudaFuncSetAttribute(gram::gram_mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, gram::SMEM);
    init = true;
  }
  SF_CHECK_ARG(((uintptr_t)probes & 7) == 0, SF_ERR_PARAM, "probe pointer array misaligned");
  // one launch per job (bi, bj); diagonal jobs feed one register set to both operands
  for (int y = 0, bi = 0; bi < nb; ++bi)
    for (int bj = bi; bj < nb; ++bj, ++y) {
      if (bi == bj)
        launch_k(gram::gram_mma_kernel<true>, dim3(nblk), dim3(gram::THREADS), gram::SMEM, st,
                 (const bf16* const*)probes, (int)K, n, y, (double*)work);
      else
        launch_k(gram::gram_mma_kernel<false>, dim3(nblk), dim3(gram::THREADS), gram::SMEM, st,
                 (const bf16* const*)probes, (int)K, n, y, (double*)work);
    }
  launch_k(gram::gram_combine_kernel, dim3(jobs), dim3(256), 0, st, (const double*)work, (int)K, nblk, out);
  return launch_status("sf_gram_bf16");
}

}  // extern "C"
