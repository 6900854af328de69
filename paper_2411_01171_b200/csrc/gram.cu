// Step Rehash similarity: the K x K Gram matrix of the K cached probe tensors in ONE pass
// over HBM (cosine_similarity, kernels.py:375-390; similarity map).
//
// G = P P^T with P the K x n matrix of probes (n = 73.7M elements at SVD-XT shape).  The
// contraction is HBM-bound (K = 25: 3.7 GB of bf16 probes per map), so every probe element is
// read exactly once, in long contiguous runs:
//  * each warp owns a contiguous element range and walks it in chunks of 256 elements; per chunk
//    and probe row the 32 lanes copy 512 contiguous bytes (cp.async, 16 B each) into the warp's
//    shared-memory stage -- one DRAM stream per row, not 64-byte scraps (the previous version
//    fed each lane's MMA fragment straight from global memory: 2.29 TB/s, 30 % of HBM in ncu;
//    this one: 0.72 ms per C3 map = 5.13 TB/s, 0.79 of the measured 6.53 TB/s copy);
//  * three stages per warp: two chunks are in flight while one is consumed;
//  * consumption: per 16-element k-step two ldmatrix.x4 per 32-row block and 8 bf16
//    mma.sync m16n8k16; on a diagonal job the A and B fragments are the same registers (B = P^T);
//  * products of bf16 values are exact; the fp32 MMA accumulators are flushed into fp64
//    registers after every chunk (256 elements), warps are combined in fixed order through
//    shared memory and blocks in fixed order by the combine kernel -- bit-reproducible.
//
// K <= 32 runs as one 32 x 32 job; larger K as one launch per pair (bi <= bj) of 32-probe
// blocks, the off-diagonal ones staging both blocks (64 rows).  Every probe must be 16-byte
// aligned (n % 8 == 0 for probes packed back to back).  Rows >= K stay zero.  The n % 256 tail
// is added in fp64 by block 0.
#include "common.cuh"

namespace sf {
namespace gram {

constexpr int CHUNK = 256;                    // elements per row per stage (512 bytes)
constexpr int STAGES = 3;
constexpr int ROWB = CHUNK * 2 + 16;          // padded row stride: the 8 rows of an ldmatrix hit distinct banks

template <bool DIAG>
struct Lay {
  static constexpr int WARPS = DIAG ? 4 : 2;             // <= 227 KB of stages per block
  static constexpr int THREADS = WARPS * 32;
  static constexpr int ROWS = DIAG ? 32 : 64;
  static constexpr int STAGE_BYTES = ROWS * ROWB;
  static constexpr int WARP_BYTES = STAGES * STAGE_BYTES;
  static constexpr int SMEM = WARPS * WARP_BYTES + 1024 * (int)sizeof(double);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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

// part[(job * gridDim.x + blockIdx.x) * 1024 + i * 32 + j]: this block's 32x32 partial of job (bi, bj)
template <bool DIAG>
__global__ void __launch_bounds__(Lay<DIAG>::THREADS, 1) gram_mma_kernel(const bf16* const* __restrict__ probes, int K, int64_t n,
                                                               int job, double* __restrict__ part) {
  using L = Lay<DIAG>;
  constexpr int WARPS = L::WARPS, THREADS = L::THREADS;
  griddep_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  const int nb = (K + 31) / 32;
  int bi, bj;
  job_of(job, nb, bi, bj);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wbuf = smem + warp * L::WARP_BYTES;
  double* comb = reinterpret_cast<double*>(smem + WARPS * L::WARP_BYTES);
  // zero every stage once: rows >= K never receive a copy
  for (int i = lane; i < L::WARP_BYTES / 16; i += 32) reinterpret_cast<uint4*>(wbuf)[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  // stage row r <-> global probe row: A block bi (rows 0-31), B block bj (rows 32-63, off-diagonal)
  const bf16* src[L::ROWS];
#pragma unroll
  for (int r = 0; r < L::ROWS; ++r) {
    const int g = (r < 32 ? bi : bj) * 32 + (r & 31);
    src[r] = g < K ? probes[g] + lane * 8 : nullptr;
  }

  const int64_t nchunks = n / CHUNK;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  const int64_t per = (nchunks + nw - 1) / nw;
  const int64_t c0 = gw * per < nchunks ? gw * per : nchunks;
  const int64_t c1 = c0 + per < nchunks ? c0 + per : nchunks;
  auto issue = [&](int64_t c, int s) {
    const uint32_t base = smem_u32(wbuf + s * L::STAGE_BYTES) + lane * 16;
#pragma unroll
    for (int r = 0; r < L::ROWS; ++r)
      if (src[r]) cp16(base + r * ROWB, src[r] + c * CHUNK);
    cp_commit();
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (c0 + s < c1) issue(c0 + s, s);
    else cp_commit();
  }

  double acc[2][4][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[m][t][e] = 0.0;
  const uint32_t lrow = (lane & 15) * ROWB + (lane >> 4) * 16;   // ldmatrix.x4 row address of this lane
  int s = 0;
  for (int64_t ch = c0; ch < c1; ++ch) {
    const int sn = s + STAGES - 1 >= STAGES ? s - 1 : s + STAGES - 1;   // (s + STAGES-1) % STAGES
    if (ch + STAGES - 1 < c1) issue(ch + STAGES - 1, sn);
    else cp_commit();
    cp_wait<STAGES - 1>();
    __syncwarp();
    float c[2][4][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) c[m][t][e] = 0.f;
    const uint32_t sb = smem_u32(wbuf + s * L::STAGE_BYTES) + lrow;
#pragma unroll 4
    for (int kk = 0; kk < CHUNK / 16; ++kk) {
      uint32_t a[2][4];                       // A rows 0-15 / 16-31 at k-step kk
      ldsm_x4(sb + kk * 32, a[0]);
      ldsm_x4(sb + 16 * ROWB + kk * 32, a[1]);
      uint32_t b[2][4];
      if (DIAG) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < 4; ++j) b[h][j] = a[h][j];
      } else {
        ldsm_x4(sb + 32 * ROWB + kk * 32, b[0]);
        ldsm_x4(sb + 48 * ROWB + kk * 32, b[1]);
      }
      // n-tile t = B rows 8t..8t+7: fragment (b0, b1) = regs {0, 2} / {1, 3} of its 16-row half
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t b0 = b[t >> 1][t & 1], b1 = b[t >> 1][2 + (t & 1)];
        mma16816(c[0][t], a[0][0], a[0][1], a[0][2], a[0][3], b0, b1);
        mma16816(c[1][t], a[1][0], a[1][1], a[1][2], a[1][3], b0, b1);
      }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[m][t][e] += (double)c[m][t][e];
    s = s + 1 == STAGES ? 0 : s + 1;
  }
  cp_wait<0>();
  // fixed-order combine of the warps: warp 0, then 1, ... (entry (m,t,e) of lane L)
  for (int w = 0; w < WARPS; ++w) {
    if (warp == w) {
      const int g = lane >> 2, q = lane & 3;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int idx = (m * 16 + g + (e >= 2 ? 8 : 0)) * 32 + t * 8 + 2 * q + (e & 1);
            comb[idx] = (w == 0 ? 0.0 : comb[idx]) + acc[m][t][e];
          }
    }
    __syncthreads();
  }
  double* out = part + ((int64_t)job * gridDim.x + blockIdx.x) * 1024;
  for (int i = threadIdx.x; i < 1024; i += THREADS) out[i] = comb[i];
  // the n % CHUNK tail elements, block 0 of every job
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

inline int blocks_per_job() { return num_sms(); }   // one block per SM (3 stages of 16.5 / 33 KB per warp)

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
  SF_CHECK_ARG(((uintptr_t)probes & 7) == 0, SF_ERR_PARAM, "probe pointer array misaligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = (K + 31) / 32, jobs = nb * (nb + 1) / 2, nblk = gram::blocks_per_job();
  static bool init = false;
  if (!init) {
    SF_CHECK_ARG(cudaFuncSetAttribute(gram::gram_mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      gram::Lay<true>::SMEM) == cudaSuccess &&
                     cudaFuncSetAttribute(gram::gram_mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          gram::Lay<false>::SMEM) == cudaSuccess,
                 SF_ERR_CUDA, "shared-memory opt-in");
    init = true;
  }
  // one launch per job (bi, bj); diagonal jobs feed one register set to both operands
  for (int y = 0, bi = 0; bi < nb; ++bi)
    for (int bj = bi; bj < nb; ++bj, ++y) {
      if (bi == bj)
        launch_k(gram::gram_mma_kernel<true>, dim3(nblk), dim3(gram::Lay<true>::THREADS), gram::Lay<true>::SMEM, st,
                 (const bf16* const*)probes, (int)K, n, y, (double*)work);
      else
        launch_k(gram::gram_mma_kernel<false>, dim3(nblk), dim3(gram::Lay<false>::THREADS), gram::Lay<false>::SMEM,
                 st,
                 (const bf16* const*)probes, (int)K, n, y, (double*)work);
    }
  launch_k(gram::gram_combine_kernel, dim3(jobs), dim3(256), 0, st, (const double*)work, (int)K, nblk, out);
  return launch_status("sf_gram_bf16");
}

}  // extern "C"
