// tcgen05 / TMEM / TMA implicit GEMM for sm_100a.
//
// One persistent, warp-specialised kernel covers every contraction of the
// sliceflow path whose channel counts are multiples of 64:
//   * conv2d 3x3 (kernels.py:181-201): A tiles are 128-pixel rectangles of one
//     frame loaded by a 4-D TMA box {64 ch, w_t, h_t, 1} per (tap, channel
//     block); the zero padding is TMA's out-of-bounds fill;
//   * temporal conv, 3 taps (kernels.py:204-225): 4-D box {64 ch, pixels,
//     frames, 1}; tap j shifts the frame coordinate by j-1, OOB frames -> 0;
//   * linear / attention projections / batched attention GEMMs (plain rows).
// B (weights, or K for S = Q K^T, or V^T) is always K-major.
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = MMA issuer (+TMEM
// allocation), warps 2..5 = epilogue (TMEM -> registers -> bias / per-frame
// bias / SiLU / residual -> global).  Shared-memory ring of STAGES
// {A 128x64, B BNx64} bf16 tiles in the canonical K-major SWIZZLE_128B layout;
// two TMEM accumulators (2 x BN fp32 columns) so the epilogue of tile t
// overlaps the mainloop of tile t+1.
#include "common.cuh"

#include <cuda.h>
#include <cstdlib>
#include <mutex>

namespace sf {
namespace tc {

constexpr int BM = 128, BK = 64;
constexpr int F32_CHUNK_BYTES = 128 * 32 * 4;   // EPI 3: one 32-column fp32 chunk of a tile
constexpr int NUM_THREADS = 320;   // warp 0 TMA, 1 MMA, 2..9 epilogue (two per TMEM lane quarter)
constexpr int EPI_W0 = 2;  // first epilogue warp

struct Params {
  int mode;
  // M tiling
  int n_inner, n_outer, T;   // PLAIN: o over n_outer (and z over batch); TCONV: o = b*T + t
  int bi, bo;                // rows of a tile = bo outer x bi inner (PLAIN/TCONV)
  int tiles_i, tiles_o, n_z; // PLAIN: tiles_o over n_outer, n_z = batch; TCONV: tiles_o over T, n_z = B
  int H, W, w_t, h_t, tiles_x, tiles_y;  // CONV (tiles_y = full h_t-row bands per frame)
  // CONV tail tiles: when H % h_t = tail_rows divides h_t, the last tail_rows rows of
  // tail_fb consecutive frames form one 128-row tile (M tiles >= n_main; maps *T)
  int64_t n_main;
  int tail_y0, tail_rows, tail_fb, n_frames;
  int64_t tiles_m;
  int tiles_n, N, BN;
  int taps, cblocks;         // K loop = taps x cblocks (64-channel blocks)
  int cin;
  int b_batched;             // B map has a batch coordinate (z)
  int collapsed;             // PLAIN rows collapsed into one contiguous range
  int a_batched;             // A map has a batch coordinate (0: one A shared by every batch)
  // epilogue
  float alpha;
  const float* bias;
  const float* rowbias;
  int64_t rowbias_stride;
  const float2* rowstats;    // folded LayerNorm (PLAIN): per row (rstd, -mean*rstd)
  const float* colvec;       // ... and per column sum_k W[n][k]
  int act;
  sf_view_t res;
  int64_t res_bstride;
  sf_view_t out;
  int64_t out_bstride;
  int out_fp32;
  // CONV, bf16 output: GroupNorm partials of the stored output, [frame][gn_splits][N] (sum, sum sq)
  // (sf_gemm_args.gn_partial; split = 64-row half of a main tile, or a frame's rows of a tail tile)
  float2* gn_part;
  int gn_splits;
};

// ---------------------------------------------------------------- PTX helpers
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
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
// ---- CTA-pair (cta_group::2) helpers ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t leader_addr(const void* ptr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(ptr)));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_4d_2sm(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1, int c2,
                                                int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// Converged-warp producer variants: every lane executes the call with warp-uniform
// operands and one elect.sync lane issues the instruction (no per-instruction
// waterfall loop, see the MMA issuer).  Only for code the whole warp runs.
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_4d_e(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                              int c3) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_e(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n}\n" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_2sm_e(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1,
                                                  int c2, int c3) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6}], [%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm_e(const CUtensorMap* map, uint32_t bar, void* dst, int c0, int c1,
                                                  int c2) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (canonical layout
// ((8,n),2):((8,SBO),1) in 16-byte units: SBO = 1024 B, LBO unused = 1).
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version = 1 (sm100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M=m, N=n
__host__ __device__ constexpr uint32_t make_idesc(int n, int m = BM) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// issue-only TMEM load (no wait); pair with tmem_wait_ld before reading r
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// per-column epilogue terms for W (32 or 16) columns starting at global column nb: alpha,
// bias, per-row bias, SiLU.  Vector loads when all W columns are in range (bias rows are
// 16-byte aligned).
template <int W = 32>
__device__ __forceinline__ void epi_columns(const Params& p, float* v, int nb, int64_t o, int64_t m = -1) {
  if (p.rowstats && m >= 0) {   // folded LayerNorm: rstd_m * (acc - mean_m * colsum_n)
    const float2 s = p.rowstats[m];
    if (nb + W <= p.N) {
      const float4* c4 = reinterpret_cast<const float4*>(p.colvec + nb);
#pragma unroll
      for (int j = 0; j < W / 4; ++j) {
        const float4 c = __ldg(c4 + j);
        v[4 * j] = fmaf(s.x, v[4 * j], s.y * c.x);
        v[4 * j + 1] = fmaf(s.x, v[4 * j + 1], s.y * c.y);
        v[4 * j + 2] = fmaf(s.x, v[4 * j + 2], s.y * c.z);
        v[4 * j + 3] = fmaf(s.x, v[4 * j + 3], s.y * c.w);
      }
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] = fmaf(s.x, v[j], s.y * (nb + j < p.N ? __ldg(p.colvec + nb + j) : 0.f));
    }
  }
  if (p.alpha != 1.f) {
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] *= p.alpha;
  }
  const bool full = nb + W <= p.N;
  if (p.bias) {
    if (full) {
      const float4* b4 = reinterpret_cast<const float4*>(p.bias + nb);
#pragma unroll
      for (int j = 0; j < W / 4; ++j) {
        const float4 b = __ldg(b4 + j);
        v[4 * j] += b.x;
        v[4 * j + 1] += b.y;
        v[4 * j + 2] += b.z;
        v[4 * j + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] += (nb + j < p.N) ? __ldg(p.bias + nb + j) : 0.f;
    }
  }
  if (p.rowbias) {
    const float* rb = p.rowbias + o * p.rowbias_stride + nb;
    if (full && ((reinterpret_cast<uintptr_t>(rb) & 15) == 0)) {
#pragma unroll
      for (int j = 0; j < W / 4; ++j) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(rb) + j);
        v[4 * j] += b.x;
        v[4 * j + 1] += b.y;
        v[4 * j + 2] += b.z;
        v[4 * j + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] += (nb + j < p.N) ? __ldg(rb + j) : 0.f;
    }
  }
  if (p.act == SF_ACT_SILU) {
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] = silu_f(v[j]);
  }
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// ---------------------------------------------------------------- tiling
struct MTile {
  int z, o0, i0;   // PLAIN/TCONV: batch/b, outer start (t0 or o0), inner start
  int f, y0, x0;   // CONV
  int tail;        // CONV: a tail tile (rows tail_y0.. of tail_fb frames starting at f)
};

template <bool CONV>
__device__ __forceinline__ MTile decode_m(const Params& p, int64_t tm) {
  MTile t{};
  if (CONV) {
    if (p.tail_rows && tm >= p.n_main) {
      const int64_t tt = tm - p.n_main;
      t.x0 = (int)(tt % p.tiles_x) * p.w_t;
      t.f = (int)(tt / p.tiles_x) * p.tail_fb;
      t.y0 = p.tail_y0;
      t.tail = 1;
    } else {
      t.x0 = (int)(tm % p.tiles_x) * p.w_t;
      int64_t r = tm / p.tiles_x;
      t.y0 = (int)(r % p.tiles_y) * p.h_t;
      t.f = (int)(r / p.tiles_y);
    }
  } else {
    t.i0 = (int)(tm % p.tiles_i) * p.bi;
    int64_t r = tm / p.tiles_i;
    t.o0 = (int)(r % p.tiles_o) * p.bo;
    t.z = (int)(r / p.tiles_o);
  }
  return t;
}

template <int BN, int STAGES, int EPI, bool PAIR = false>
struct SmemLayout {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;   // a pair stages half of B per CTA
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // epilogue staging tile [128 rows][BN] bf16 (residual in, output out), row-major
  static constexpr int OUT_TILE = BM * BN * 2;
  // EPI staging buffers: 0 = direct stores; 1/2 = bf16 tiles; 3 = two 128 x 32 fp32 chunks (SW128)
  static constexpr int OUT_BYTES = EPI == 3 ? 4 * F32_CHUNK_BYTES : EPI * OUT_TILE;
  static constexpr int TOTAL = 1024 /*align slack*/ + STAGES * STAGE_BYTES + OUT_BYTES + 512 /*barriers*/;
};

// TMEM accumulator buffers (<= TC_NACC_MAX BN-column tiles in the 512 columns).  3-4 buffers
// measured neutral (<= 2 % on K = 320 GEMMs): the MMA warp gets its buffer back right after the
// commit (tools/gemm_trace.py); it waits on operand stages, i.e. the L2 throughput cap
#ifndef TC_NACC_MAX
#define TC_NACC_MAX 2
#endif
template <int BN>
constexpr int nacc() {
  return 512 / BN >= TC_NACC_MAX ? TC_NACC_MAX : (512 / BN < 2 ? 2 : 512 / BN);
}

// -DTC_TRACE (tuning builds only): SM-clock stamps of CTA 0's pipeline events, per role
#ifdef TC_TRACE
__device__ unsigned long long g_tc_trace[4][4096];
__device__ unsigned int g_tc_trace_n[4];
#define TC_TR(role, code)                                                                 \
  do {                                                                                    \
    if (blockIdx.x == 0) {                                                                \
      const unsigned i_ = g_tc_trace_n[role]++;                                           \
      if (i_ < 4096) g_tc_trace[role][i_] = ((unsigned long long)clock64() << 4) | (code); \
    }                                                                                     \
  } while (0)
#else
#define TC_TR(role, code) \
  do {                    \
  } while (0)
#endif

// Per-(frame, split, channel) (sum, sum sq) of one staged bf16 half-tile (128 rows x HC columns,
// row-major): thread t sums column pair t % 64 over the 64 rows of half t / 64 -- one frame in a
// main tile; in a tail tile the half holds 64 / per whole frame segments of per (16/32/64) rows.
// Rows r = 4i + u go to accumulator u (four independent chains), combined as (0+1)+(2+3); the
// pass kernel (elementwise.cu conv_gn_partials_kernel) uses the same order.
template <int HC>
__device__ __forceinline__ void gn_tile_partials(const Params& p, const MTile& mt, const uint8_t* hbuf, int hn0,
                                                 int t) {
  const int pair = t & 63, rh = t >> 6;
  if (2 * pair >= HC || hn0 + 2 * pair >= p.N) return;
  const int lg = __ffs(p.w_t) - 1;                      // w_t is a power of two
  const int per = mt.tail ? p.tail_rows * p.w_t : 64;   // rows per frame segment (<= 64)
  for (int s0 = rh * 64; s0 < rh * 64 + 64; s0 += per) {
    const int fr = mt.tail ? mt.f + s0 / per : mt.f;
    if (fr >= p.n_frames) break;
    float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
    float q0[4] = {0.f, 0.f, 0.f, 0.f}, q1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r = s0; r < s0 + per; r += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = (mt.tail ? r - s0 : r) + u;
        const int y = mt.y0 + (rr >> lg), x = mt.x0 + (rr & (p.w_t - 1));
        const float2 f = __bfloat1622float2(*reinterpret_cast<const bf162*>(hbuf + (r + u) * (HC * 2) + pair * 4));
        if (y < p.H && x < p.W) {
          a0[u] += f.x;
          q0[u] = fmaf(f.x, f.x, q0[u]);
          a1[u] += f.y;
          q1[u] = fmaf(f.y, f.y, q1[u]);
        }
      }
    }
    const int split = mt.tail ? 2 * p.tiles_x * p.tiles_y + (mt.x0 >> lg)
                              : 2 * ((mt.y0 / p.h_t) * p.tiles_x + (mt.x0 >> lg)) + rh;
    *reinterpret_cast<float4*>(p.gn_part + ((int64_t)fr * p.gn_splits + split) * p.N + hn0 + 2 * pair) =
        make_float4((a0[0] + a0[1]) + (a0[2] + a0[3]), (q0[0] + q0[1]) + (q0[2] + q0[3]),
                    (a1[0] + a1[1]) + (a1[2] + a1[3]), (q1[0] + q1[1]) + (q1[2] + q1[3]));
  }
}

// PAIR: CTA pairs (cluster of 2) run tcgen05.mma.cta_group::2 with M = 256:
// CTA rank r owns M-tile 2*pair + r (its A rows, TMEM accumulator and epilogue)
// and stages rows [r*BN/2, (r+1)*BN/2) of the B tile; the leader (rank 0)
// issues every MMA and its commits arrive on both CTAs' barriers.
// CONV: 3x3-conv instance (2-D frame tiles, tail tiles, tap-shifted boxes); the plain / temporal
// instance carries none of that code (measured: up to 5 % on short-K GEMMs, profiles finding 20)
template <int BN, int STAGES, int EPI, bool PAIR, bool CONV>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapR,
                   const __grid_constant__ CUtensorMap mapO, const __grid_constant__ CUtensorMap mapAT,
                   const __grid_constant__ CUtensorMap mapRT, const __grid_constant__ CUtensorMap mapOT) {
  using L = SmemLayout<BN, STAGES, EPI, PAIR>;
  constexpr bool TMA_EPI = EPI == 1 || EPI == 2;   // bf16 staging + TMA store (EPI 3: fp32 chunks)
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by offsetting the shared array itself (a uintptr_t round trip loses
  // the shared address space: every C++ staging access became a generic LD/ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint8_t* sOut = smem + STAGES * L::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + L::OUT_BYTES);
  uint64_t* empty = full + STAGES;
  constexpr int NACC = nacc<BN>();
  uint64_t* tfull = empty + STAGES;   // [NACC]
  uint64_t* tempty = tfull + NACC;    // [NACC]
  uint64_t* res_full = tempty + NACC; // [2 buffers][2 halves] residual half-tile landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(res_full + 4);
  const bool has_res = TMA_EPI && p.res.ptr != nullptr;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t TMEM_COLS = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128
                                 : (NACC * BN <= 256) ? 256 : 512;
  static_assert(NACC * BN <= 512, "TMEM accumulators");

  if (warp == 0 && lane == 0) {
    prefetch_map(&mapA);
    prefetch_map(&mapB);
    if (p.tail_rows) prefetch_map(&mapAT);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < NACC; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], PAIR ? 16 : 8);  // one arrive per epilogue warp (of both CTAs)
    }
    for (int b = 0; b < 4; ++b) mbar_init(&res_full[b], 1);
    if (TMA_EPI || EPI == 3) {
      prefetch_map(&mapO);
      if (has_res) prefetch_map(&mapR);
      if (p.tail_rows) {
        prefetch_map(&mapOT);
        if (has_res) prefetch_map(&mapRT);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue (barriers, TMEM) done without touching global data: now wait for the
  // producing kernel (PDL).  The next kernel is released (griddep_trigger) once this CTA's
  // producer has issued its last load, so its prologue overlaps our last tiles' MMAs/epilogues.
  griddep_wait();

  const int kiters = p.taps * p.cblocks;
  // tile walk: a pair walks pair-tiles (two adjacent M-tiles x one N-tile)
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int64_t tiles_mw = PAIR ? (p.tiles_m + 1) / 2 : p.tiles_m;
  const int64_t n_tiles = tiles_mw * p.tiles_n;
  const int64_t t_first = PAIR ? blockIdx.x / 2 : blockIdx.x;
  const int64_t t_step = PAIR ? gridDim.x / 2 : gridDim.x;
  auto my_tm = [&](int64_t tile) -> int64_t {
    const int64_t tw = tile / p.tiles_n;
    return PAIR ? 2 * tw + rank : tw;
  };

  if (warp == 0) {
    // ================= TMA producer (whole warp converged, elect.sync issue) =================
    {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tcount = 0;
      for (int64_t tile = t_first; tile < n_tiles; tile += t_step, ++tcount) {
        const int64_t tm = my_tm(tile);
        const int n0 = (int)(tile % p.tiles_n) * BN;
        const MTile mt = decode_m<CONV>(p, tm);
        for (int it = 0; it < kiters; ++it) {
          const int tap = it / p.cblocks, cb = it % p.cblocks;
          mbar_wait(&empty[stage], phase ^ 1);
          if (lane == 0) TC_TR(0, 1);
          void* dA = sA + stage * L::A_BYTES;
          void* dB = sB + stage * L::B_BYTES;
          if constexpr (PAIR) {
            // my A tile + my half of B, completion bytes counted on the leader's barrier
            if (leader) mbar_expect_tx_e(&full[stage], 2 * L::STAGE_BYTES);
            const uint32_t fb = leader_addr(&full[stage]);
            if (CONV)
              tma_load_4d_2sm_e(mt.tail ? &mapAT : &mapA, fb, dA, cb * BK, mt.x0 + tap % 3 - 1, mt.y0 + tap / 3 - 1,
                              mt.f);
            else if (p.mode == SF_GEMM_TCONV3)
              tma_load_4d_2sm_e(&mapA, fb, dA, cb * BK, mt.i0, mt.o0 + tap - 1, mt.z);
            else
              tma_load_4d_2sm_e(&mapA, fb, dA, cb * BK, mt.i0, mt.o0, p.a_batched ? mt.z : 0);
            tma_load_3d_2sm_e(&mapB, fb, dB, tap * p.cin + cb * BK, n0 + (int)rank * (BN / 2), p.b_batched ? mt.z : 0);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          mbar_expect_tx_e(&full[stage], L::STAGE_BYTES);
          if (CONV) {
            tma_load_4d_e(mt.tail ? &mapAT : &mapA, &full[stage], dA, cb * BK, mt.x0 + tap % 3 - 1,
                        mt.y0 + tap / 3 - 1, mt.f);
          } else if (p.mode == SF_GEMM_TCONV3) {
            tma_load_4d_e(&mapA, &full[stage], dA, cb * BK, mt.i0, mt.o0 + tap - 1, mt.z);
          } else {
            tma_load_4d_e(&mapA, &full[stage], dA, cb * BK, mt.i0, mt.o0, p.a_batched ? mt.z : 0);
          }
          tma_load_3d_e(&mapB, &full[stage], dB, tap * p.cin + cb * BK, n0, p.b_batched ? mt.z : 0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // drain: the MMA's release of every ring slot (a tcgen05.commit, multicast into this CTA's
      // barrier in PAIR mode) must have landed before the CTA retires -- an arrive landing later
      // would write into the shared memory of whichever CTA the SM hosts next
      for (int s = 0; s < STAGES; ++s) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    griddep_trigger();
  } else if (warp == 1) {
    // ================= MMA issuer =================
    // whole warp converged; each tcgen05 instruction is issued by one elect.sync lane, so the
    // descriptors are warp-uniform and ptxas emits no per-MMA waterfall loop
    if (leader) {
      constexpr uint32_t idesc = make_idesc(BN, PAIR ? 2 * BM : BM);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t tile = t_first; tile < n_tiles; tile += t_step) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        if (lane == 0) TC_TR(1, 2);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int it = 0; it < kiters; ++it) {
          mbar_wait(&full[stage], phase);
          if (lane == 0) TC_TR(1, 3);
          tc_fence_after();
          const uint64_t ad = make_sdesc(smem_u32(sA + stage * L::A_BYTES));
          const uint64_t bd = make_sdesc(smem_u32(sB + stage * L::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 B along K inside the 128 B swizzle atom = +2 in the 16-byte address field
            if (PAIR) umma_f16_pair(d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (it | k) != 0);
            else umma_f16(d, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (it | k) != 0);
          }
          if (PAIR) umma_commit_pair(&empty[stage]);
          else umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (PAIR) umma_commit_pair(&tfull[acc]);
        else umma_commit(&tfull[acc]);
        if (lane == 0) TC_TR(1, 4);
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ================= epilogue =================
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int eh = (warp - EPI_W0) >> 2;    // column half: 32-column chunks eh, eh+2, eh+4, ...
    const int row = q * 32 + lane;          // accumulator row == TMEM lane
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t tcount = 0;
    const uint32_t tempty_l = PAIR ? leader_addr(&tempty[0]) : 0;
    int chunk = 0;   // EPI 3: this half's chunk count over all its tiles (staging buffer = chunk & 1)
    for (int64_t tile = t_first; tile < n_tiles; tile += t_step, ++tcount) {
      const int64_t tm = my_tm(tile);
      const int n0 = (int)(tile % p.tiles_n) * BN;
      const MTile mt = decode_m<CONV>(p, tm);
      const bool phantom = tm >= p.tiles_m;   // odd tile count: the pair's second tile is empty
      // output row of this thread
      bool valid;
      int64_t o, i;
      int z = 0;
      if (CONV) {
        // main tile: rows (y, x) of one frame; tail tile: (frame, y, x) over tail_fb frames
        const int per = mt.tail ? p.tail_rows * p.w_t : BM;
        const int fr = mt.f + row / per, rr = row % per;
        const int y = mt.y0 + rr / p.w_t, x = mt.x0 + rr % p.w_t;
        valid = y < p.H && x < p.W && fr < p.n_frames;
        o = fr;
        i = (int64_t)y * p.W + x;
      } else {
        const int oo = mt.o0 + row / p.bi, ii = mt.i0 + row % p.bi;
        if (p.mode == SF_GEMM_TCONV3) {
          valid = oo < p.T && ii < p.n_inner;
          o = (int64_t)mt.z * p.T + oo;
        } else {
          valid = oo < p.n_outer && ii < p.n_inner;
          o = oo;
          z = mt.z;
        }
        i = ii;
      }
      valid = valid && !phantom;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if constexpr (EPI == 3) {
        // fp32 output through two 16 KB staging chunks (128 rows x 32 cols, 128-byte swizzle:
        // a thread's row lands in a different bank group than its 7 neighbours), one TMA
        // store per chunk; a chunk buffer is refilled once its store from two chunks ago is read
        // each column half (4 warps) stages its own chunks: buffers 2*eh + (chunk & 1), its own
        // leader and named barrier (2 + eh).  The chunk count runs across tiles: with BN = 64
        // a half has one chunk per tile, and a per-tile count would refill the buffer whose
        // store (the previous tile's) wait_group.read 1 leaves in flight -- corrupted rows
        // whenever that store's shared-memory read was slow (concurrent streams: profiles
        // finding 30)
        const bool store_leader = warp == EPI_W0 + 4 * eh && lane == 0;
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int c = eh * 32; c < BN; c += 64, ++chunk) {
          float v[32];
          tmem_ld32(tbase + c, v);
          const int nb = n0 + c;
          if (p.rowstats && valid) {
            const float2 s = p.rowstats[o * p.n_inner + i];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fmaf(s.x, v[j], s.y * ((nb + j < p.N) ? __ldg(p.colvec + nb + j) : 0.f));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
          if (p.bias) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += (nb + j < p.N) ? __ldg(p.bias + nb + j) : 0.f;
          }
          if (p.rowbias) {
            const float* rb = p.rowbias + o * p.rowbias_stride + nb;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += (nb + j < p.N) ? __ldg(rb + j) : 0.f;
          }
          if (p.act == SF_ACT_SILU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = silu_f(v[j]);
          }
          uint8_t* buf = sOut + (2 * eh + (chunk & 1)) * F32_CHUNK_BYTES;
          if (store_leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (eh) asm volatile("bar.sync 3, 128;" ::: "memory");
          else asm volatile("bar.sync 2, 128;" ::: "memory");
          uint8_t* srow = buf + row * 128;
          const int sw = row & 7;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            *reinterpret_cast<float4*>(srow + ((u ^ sw) << 4)) =
                make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (eh) asm volatile("bar.sync 3, 128;" ::: "memory");
          else asm volatile("bar.sync 2, 128;" ::: "memory");
          if (store_leader && nb < p.N) {
            if (CONV)
              tma_store_4d(mt.tail ? &mapOT : &mapO, buf, nb, mt.x0, mt.y0, mt.f);
            else
              tma_store_4d(&mapO, buf, nb, mt.i0, mt.o0, mt.z);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) arrive_remote(tempty_l + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      if constexpr (TMA_EPI) {
        // The two column halves (4 warps each, one per TMEM lane quarter) run independently:
        // each owns a contiguous BN/2-column staging sub-tile, its residual barrier, its
        // leader (residual prefetch + TMA store) and a 128-thread named barrier, so neither
        // half waits for the other before its store.
        constexpr int HC = BN / 2;                    // columns per half
        constexpr int HALF_BYTES = BM * HC * 2;
        const bool hleader = warp == EPI_W0 + 4 * eh && lane == 0;
        const int ob = EPI == 2 ? (int)(tcount & 1) : 0;
        const uint32_t use = EPI == 2 ? (tcount >> 1) : tcount;
        uint8_t* hbuf = sOut + ob * L::OUT_TILE + eh * HALF_BYTES;
        const int hn0 = n0 + eh * HC;
        uint64_t* rf = &res_full[ob * 2 + eh];
        auto load_res_half = [&](uint64_t* bar, uint8_t* dst, int col, const MTile& m) {
          if (CONV)
            tma_load_4d(m.tail ? &mapRT : &mapR, bar, dst, col, m.x0, m.y0, m.f);
          else
            tma_load_4d(&mapR, bar, dst, col, m.i0, m.o0, m.z);
        };
        auto half_sync = [&]() {
          if (eh) asm volatile("bar.sync 3, 128;" ::: "memory");
          else asm volatile("bar.sync 2, 128;" ::: "memory");
        };
        if (EPI == 1) {
          // single staging buffer: my previous store must have drained it; then fetch my residual
          if (hleader) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (has_res) {
              mbar_expect_tx(rf, HALF_BYTES);
              load_res_half(rf, hbuf, hn0, mt);
            }
          }
          half_sync();
        } else if (has_res && hleader) {
          // double staging: the first tile's residual now; every epilogue then prefetches the
          // next tile's residual into the other buffer once that buffer's store has been read
          if (tcount == 0) {
            mbar_expect_tx(rf, HALF_BYTES);
            load_res_half(rf, hbuf, hn0, mt);
          }
          const int64_t nt = tile + t_step;
          if (nt < n_tiles) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            const MTile nm = decode_m<CONV>(p, my_tm(nt));
            const int nn0 = (int)(nt % p.tiles_n) * BN + eh * HC;
            uint64_t* rfn = &res_full[(ob ^ 1) * 2 + eh];
            mbar_expect_tx(rfn, HALF_BYTES);
            load_res_half(rfn, sOut + (ob ^ 1) * L::OUT_TILE + eh * HALF_BYTES, nn0, nm);
          }
        }
        mbar_wait(&tfull[acc], acc_phase);
        if (hleader) TC_TR(2 + eh, 5);
        tc_fence_after();
        if (has_res) mbar_wait(rf, use & 1);
        uint8_t* srow = hbuf + row * (HC * 2);
        const int64_t srow_m = (p.rowstats && valid) ? o * p.n_inner + i : -1;   // folded-LN row
        auto finish32 = [&](int c) {
          float v[32];
          tmem_ld32(tbase + eh * HC + c, v);
          epi_columns<32>(p, v, hn0 + c, o, srow_m);
          bf16x8* sp = reinterpret_cast<bf16x8*>(srow + c * 2);
          if (has_res) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float f[8];
              unpack8(sp[j], f);
#pragma unroll
              for (int e = 0; e < 8; ++e) v[j * 8 + e] += f[e];
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) sp[j] = pack8(v + 8 * j);
        };
#pragma unroll 1
        for (int c = 0; c + 32 <= HC; c += 32) finish32(c);
        if constexpr (HC % 32 == 16) {
          const int c = HC - 16;
          float v[16];
          tmem_ld16(tbase + eh * HC + c, v);
          epi_columns<16>(p, v, hn0 + c, o, srow_m);
          bf16x8* sp = reinterpret_cast<bf16x8*>(srow + c * 2);
          if (has_res) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              float f[8];
              unpack8(sp[j], f);
#pragma unroll
              for (int e = 0; e < 8; ++e) v[j * 8 + e] += f[e];
            }
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) sp[j] = pack8(v + 8 * j);
        }
        // accumulator free for the tile after next
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR) arrive_remote(tempty_l + acc * 8);
          else mbar_arrive(&tempty[acc]);
        }
        if (hleader) TC_TR(2 + eh, 6);
        // my half-tile complete -> my leader stores it with TMA (OOB rows/cols are clipped)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        half_sync();
        if (hleader) {
          if (hn0 < p.N) {
            if (CONV)
              tma_store_4d(mt.tail ? &mapOT : &mapO, hbuf, hn0, mt.x0, mt.y0, mt.f);
            else
              tma_store_4d(&mapO, hbuf, hn0, mt.i0, mt.o0, mt.z);
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if constexpr (CONV) {
          // GroupNorm partials of the next op (res.norm2 reads this conv's output, unet.py:191-193)
          // from the staged bf16 half-tile -- the exact values stored -- while the TMA store reads
          // it too: thread = (64-row half, column pair); fixed order, no atomics.  The buffer is
          // next written after the next tile's opening half_sync, except by EPI 1's residual load,
          // which its leader issues before that barrier: then wait for every reader here
          if (p.gn_part != nullptr && !phantom) {
            gn_tile_partials<HC>(p, mt, hbuf, hn0, row);
            if (EPI == 1 && has_res) half_sync();
          }
        }
        if (hleader) {
          // the other buffer's store (tile t-1) must drain before it is refilled
          if (EPI == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          TC_TR(2 + eh, 7);
        }
        if (EPI == 2) half_sync();
        if (hleader) TC_TR(2 + eh, 8);
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = eh * 32; c < BN; c += 64) {
        float v[32];
        tmem_ld32(tbase + c, v);
        const int nb = n0 + c;
        if (valid && nb < p.N) {
          const int ncols = min(32, p.N - nb);
          if (p.rowstats) {
            const float2 s = p.rowstats[o * p.n_inner + i];
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncols) v[j] = fmaf(s.x, v[j], s.y * __ldg(p.colvec + nb + j));
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] *= p.alpha;
          if (p.bias) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncols) v[j] += __ldg(p.bias + nb + j);
          }
          if (p.rowbias) {
            const float* rb = p.rowbias + o * p.rowbias_stride + nb;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < ncols) v[j] += __ldg(rb + j);
          }
          if (p.act == SF_ACT_SILU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = silu_f(v[j]);
          }
          if (p.res.ptr) {
            const bf16* rr = reinterpret_cast<const bf16*>(p.res.ptr) + (int64_t)z * p.res_bstride +
                             (o * p.res.ostride + i) * p.res.ld + nb;
            if (ncols == 32) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float f[8];
                unpack8(reinterpret_cast<const bf16x8*>(rr)[j], f);
#pragma unroll
                for (int e = 0; e < 8; ++e) v[j * 8 + e] += f[e];
              }
            } else {
              for (int j = 0; j < ncols; ++j) v[j] += __bfloat162float(rr[j]);
            }
          }
          if (p.out_fp32) {
            float* dst = reinterpret_cast<float*>(p.out.ptr) + (int64_t)z * p.out_bstride +
                         (o * p.out.ostride + i) * p.out.ld + nb;
            if (ncols == 32) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                reinterpret_cast<float4*>(dst)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            } else {
              for (int j = 0; j < ncols; ++j) dst[j] = v[j];
            }
          } else {
            bf16* dst = reinterpret_cast<bf16*>(p.out.ptr) + (int64_t)z * p.out_bstride +
                        (o * p.out.ostride + i) * p.out.ld + nb;
            if (ncols == 32) {
#pragma unroll
              for (int j = 0; j < 4; ++j) reinterpret_cast<bf16x8*>(dst)[j] = pack8(v + 8 * j);
            } else {
              for (int j = 0; j < ncols; ++j) dst[j] = __float2bfloat16(v[j]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) arrive_remote(tempty_l + acc * 8);
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  // every thread that issued bulk (TMA) stores -- the leader of each column half -- waits for them
  // before the CTA retires: its shared-memory staging may belong to another kernel's CTA right
  // after (a concurrent stream), so a store still reading it would write that CTA's bytes
  if (EPI > 0 && (warp == EPI_W0 || warp == EPI_W0 + 4) && lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static bool encode(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
                   const uint32_t* box, bool swizzle = true, bool fp32 = false) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[5], s[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
  }
  for (int i = 0; i < rank - 1; ++i) s[i] = strides_bytes[i];
  CUresult r = fn(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                  const_cast<void*>(base), d, s, b, e,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int pick_bn(int N) {
  if (N % 256 == 0 && N >= 1024) return 256;
  if (N % 160 == 0) return 160;
  if (N % 128 == 0) return 128;
  if (N <= 64) return 64;
  return 128;
}

// Tile width and CTA pairing from a wave-quantisation model: a persistent grid
// of `slots` CTAs (pairs) runs ceil(tiles / slots) rounds, each as long as one
// tile's per-CTA work (128 x BN x K) times a per-width efficiency factor.
// Pairs and wide tiles win unless they cost whole extra rounds.
// wide_ok: the 192 / 224 column tiles (CTA pairs, bf16 output, long K) may be used; their
// last N tile may be partial (OOB B rows load as zeros, stores clip)
static bool choose_tiling(int N, int64_t tiles_m, bool pair_ok, bool wide_ok, int* bn) {
  // per-unit-work cost by tile width, measured on B200 conv shapes (L0 conv, N = 128..1024):
  // narrower tiles move more operand bytes per flop (N=160 ~1.15x, N=128 ~1.3x of N=256)
  auto eff = [](int b) {
    return b >= 256 ? 1.0 : b == 224 ? 1.04 : b == 192 ? 1.08 : b == 160 ? 1.15 : b == 128 ? 1.3 : 1.6;
  };
  const int sms = num_sms();
  int cands[6], nc = 0;
  cands[nc++] = *bn;
  if (N % 256 == 0 && N >= 1024 && *bn != 256) cands[nc++] = 256;
  if (N % 160 == 0 && *bn != 160) cands[nc++] = 160;
  if (N % 128 == 0 && *bn != 128) cands[nc++] = 128;
  if (wide_ok && pair_ok && N > 256) {
    cands[nc++] = 224;
    cands[nc++] = 192;
  }
  static const char* bn_env = getenv("SF_GEMM_BN");   // tuning override (same-box A/B)
  if (bn_env) {
    const int f = atoi(bn_env);
    if (f == 256 || f == 160 || f == 128 || f == 64 || ((f == 224 || f == 192) && wide_ok && pair_ok)) {
      *bn = f;
      return pair_ok;
    }
  }
  double best = 1e300;
  bool best_pair = pair_ok;
  int best_bn = *bn;
  for (int pass = 0; pass < 2; ++pass) {
    const bool pr = pass == 0;
    if (pr && !pair_ok) continue;
    for (int c = 0; c < nc; ++c) {
      const int b = cands[c];
      if (!pr && (b == 224 || b == 192)) continue;
      const int64_t tn = (N + b - 1) / b;
      const int64_t tiles = (pr ? (tiles_m + 1) / 2 : tiles_m) * tn;
      const int64_t slots = pr ? sms / 2 : sms;
      const double cost = (double)((tiles + slots - 1) / slots) * b * eff(b) * (pr ? 1.0 : 1.06);
      if (cost < best * 0.999) {
        best = cost;
        best_pair = pr;
        best_bn = b;
      }
    }
  }
  *bn = best_bn;
  return best_pair;
}

// every tensor map a launch needs (the *T maps: conv tail tiles, see Params)
struct Maps {
  CUtensorMap a, b, r, o, at, rt, ot;
};

}  // namespace tc

#ifdef TC_TRACE
// tuning builds only (not in the public header): copy out and reset CTA 0's event trace
extern "C" int32_t sf_debug_gemm_trace(unsigned long long* host, int32_t n_per_role, uint32_t* counts) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(counts, tc::g_tc_trace_n, sizeof(unsigned) * 4);
  for (int r = 0; r < 4; ++r)
    cudaMemcpyFromSymbol(host + (size_t)r * n_per_role, tc::g_tc_trace, sizeof(unsigned long long) * n_per_role,
                         sizeof(unsigned long long) * 4096 * r);
  const unsigned zero[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbol(tc::g_tc_trace_n, zero, sizeof(zero));
  return 0;
}
#endif

bool gemm_tc_supported(const sf_gemm_args& a) {
  if (!a.w_kmajor) return false;
  if (a.cin % 64 && !(a.mode == SF_GEMM_PLAIN && a.cin > 64 && a.cin % 8 == 0)) return false;
  if (a.out_fp32 == 0 && (a.out.ld % 8 || !aligned16(a.out.ptr))) return false;
  if (a.out_fp32 == 0 && ((a.out.ostride * a.out.ld * 2) % 16 || (a.out_bstride * 2) % 16)) return false;
  if (a.res.ptr && ((a.res.ostride * a.res.ld * 2) % 16 || (a.res_bstride * 2) % 16)) return false;
  if (a.res.ptr && (a.res.ld % 8 || !aligned16(a.res.ptr))) return false;
  if (a.mode == SF_GEMM_CONV3X3 && a.batch != 1) return false;
  if (a.mode == SF_GEMM_TCONV3 && a.batch != 1) return false;
  // strides must be multiples of 16 bytes for TMA
  if ((a.a.ostride * a.a.ld * 2) % 16 || (a.a_bstride * 2) % 16 || (a.w_bstride * 2) % 16) return false;
  return tc::encode_fn() != nullptr;
}

template <int BN, int STAGES, int EPI, bool PAIR, bool CONV>
static sf_status launch_one(const tc::Params& p, const tc::Maps& m, cudaStream_t st) {
  constexpr int smem = tc::SmemLayout<BN, STAGES, EPI, PAIR>::TOTAL;
  static_assert(smem <= 232448, "shared memory budget");
  static bool init = false;
  auto kern = tc::tc_gemm_kernel<BN, STAGES, EPI, PAIR, CONV>;
  if (!init) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  if (!PAIR) {
    int64_t tiles = p.tiles_m * p.tiles_n;
    int grid = (int)(tiles < num_sms() ? tiles : num_sms());
    launch_k(kern, dim3(grid), dim3(tc::NUM_THREADS), smem, st, p, m.a, m.b, m.r, m.o, m.at, m.rt, m.ot);
    return launch_status("sf_gemm(tcgen05)");
  }
  const int64_t pair_tiles = (p.tiles_m + 1) / 2 * p.tiles_n;
  const int64_t max_pairs = num_sms() / 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * (pair_tiles < max_pairs ? pair_tiles : max_pairs)), 1, 1);
  cfg.blockDim = dim3(tc::NUM_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, p, m.a, m.b, m.r, m.o, m.at, m.rt, m.ot);
  return launch_status("sf_gemm(tcgen05 pair)");
}

template <int BN, int STAGES, int EPI, bool PAIR = false>
static sf_status launch_cfg(const tc::Params& p, const tc::Maps& m, cudaStream_t st) {
  return p.mode == SF_GEMM_CONV3X3 ? launch_one<BN, STAGES, EPI, PAIR, true>(p, m, st)
                                   : launch_one<BN, STAGES, EPI, PAIR, false>(p, m, st);
}

// Output / residual maps share the M tiling of A: box {BN cols, tile rows}.
static bool encode_rows_map(CUtensorMap* m, const sf_gemm_args& a, const tc::Params& p, const sf_view_t& v,
                            int64_t bstride, int BN, bool tail = false, bool fp32 = false) {
  // fp32 (EPI 3): 32-column boxes in the 128-byte swizzle; bf16: one BN-wide unswizzled box
  const uint64_t es = fp32 ? 4 : 2, ld = (uint64_t)v.ld;
  const uint32_t bw = fp32 ? 32u : (uint32_t)(BN / 2);   // bf16: one box per column half
  if (a.mode == SF_GEMM_CONV3X3) {
    uint64_t dims[4] = {(uint64_t)a.N, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.n_outer};
    uint64_t str[3] = {ld * es, (uint64_t)a.W * ld * es,
                       (uint64_t)(v.ostride ? v.ostride : (int64_t)a.H * a.W) * ld * es};
    uint32_t box[4] = {bw, (uint32_t)p.w_t, (uint32_t)(tail ? p.tail_rows : p.h_t), (uint32_t)(tail ? p.tail_fb : 1)};
    return tc::encode(m, v.ptr, 4, dims, str, box, fp32, fp32);
  }
  uint64_t dims[4], str[3];
  dims[0] = (uint64_t)a.N;
  dims[1] = (uint64_t)p.n_inner;
  str[0] = ld * es;
  const int64_t ost = p.collapsed ? p.n_inner : (v.ostride ? v.ostride : p.n_inner);
  str[1] = (uint64_t)ost * ld * es;
  if (a.mode == SF_GEMM_TCONV3) {
    dims[2] = (uint64_t)p.T;
    dims[3] = (uint64_t)p.n_z;
    str[2] = (uint64_t)p.T * str[1];
  } else {
    dims[2] = (uint64_t)p.n_outer;
    dims[3] = (uint64_t)p.n_z;
    str[2] = p.n_z > 1 ? (uint64_t)bstride * es : (uint64_t)p.n_outer * str[1];
  }
  uint32_t box[4] = {bw, (uint32_t)p.bi, (uint32_t)p.bo, 1};
  return tc::encode(m, v.ptr, 4, dims, str, box, fp32, fp32);
}

sf_status gemm_tc_launch(const sf_gemm_args& a, cudaStream_t st) {
  using namespace tc;
  Params p{};
  p.mode = a.mode;
  p.N = a.N;
  p.cin = a.cin;
  // plain GEMMs may end in a partial K block (e.g. P.V over 144 tokens): the A / B tensor maps
  // stop at cin, so the block's tail loads as zeros (TMA OOB fill) and adds nothing
  p.cblocks = (a.cin + BK - 1) / BK;
  p.taps = a.mode == SF_GEMM_PLAIN ? 1 : (a.mode == SF_GEMM_CONV3X3 ? 9 : 3);
  p.alpha = a.alpha;
  p.bias = a.bias;
  p.rowbias = a.rowbias;
  p.rowbias_stride = a.rowbias_stride;
  p.rowstats = reinterpret_cast<const float2*>(a.rowstats);
  p.colvec = a.colvec;
  p.act = a.act;
  p.res = a.res;
  p.res_bstride = a.res_bstride;
  p.out = a.out;
  p.out_bstride = a.out_bstride;
  p.out_fp32 = a.out_fp32;
  CUtensorMap ma, mb, mat;
  const uint64_t es = 2;
  // CTA pairs (cta_group::2, M = 256) whenever there are two M-tiles to pair up;
  // SF_GEMM_PAIR=0 forces single-CTA tiles (A/B runs)
  static const char* pair_env = getenv("SF_GEMM_PAIR");
  bool pair = !(pair_env && pair_env[0] == '0') && !(a.backend & SF_GEMM_NO_PAIR);
  const uint64_t ld = (uint64_t)a.a.ld;
  if (a.mode == SF_GEMM_CONV3X3) {
    p.H = a.H;
    p.W = a.W;
    const ConvTiling ct = conv_tiling(a.H, a.W);
    p.w_t = ct.w_t;
    p.h_t = ct.h_t;
    p.tiles_x = ct.tiles_x;
    p.tiles_y = (a.H + p.h_t - 1) / p.h_t;
    p.tiles_m = (int64_t)p.tiles_x * p.tiles_y * a.n_outer;
    uint64_t dims[4] = {(uint64_t)a.cin, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.n_outer};
    uint64_t str[3] = {ld * es, (uint64_t)a.W * ld * es, (uint64_t)a.a.ostride * ld * es};
    uint32_t box[4] = {BK, (uint32_t)p.w_t, (uint32_t)p.h_t, 1};
    if (a.n_outer == 1) str[2] = (uint64_t)a.H * a.W * ld * es;
    SF_CHECK_ARG(encode(&ma, a.a.ptr, 4, dims, str, box), SF_ERR_CUDA, "tensor map A (conv)");
    // tail tiles: the H % h_t leftover rows of h_t / rem consecutive frames as one tile
    // (e.g. 9x16 frames: 8-row tiles + the 9th row of 8 frames instead of 25 near-empty tiles)
    p.n_frames = a.n_outer;
    p.n_main = p.tiles_m;
    const int rem = a.H % p.h_t;
    if (ct.tail_rows) {
      const int fb = ct.tail_fb;
      uint32_t tbox[4] = {BK, (uint32_t)p.w_t, (uint32_t)rem, (uint32_t)fb};
      if (encode(&mat, a.a.ptr, 4, dims, str, tbox)) {
        p.tail_rows = rem;
        p.tail_fb = fb;
        p.tiles_y = a.H / p.h_t;
        p.tail_y0 = p.tiles_y * p.h_t;
        p.n_main = (int64_t)p.tiles_x * p.tiles_y * a.n_outer;
        p.tiles_m = p.n_main + (int64_t)p.tiles_x * ((a.n_outer + fb - 1) / fb);
      }
    }
    if (a.gn_partial) {
      p.gn_part = reinterpret_cast<float2*>(a.gn_partial);
      p.gn_splits = 2 * p.tiles_x * p.tiles_y + (p.tail_rows ? p.tiles_x : 0);
      SF_CHECK_ARG(p.gn_splits == ct.gn_splits(), SF_ERR_CUDA, "conv tiling disagrees with sf_conv_gn_splits");
    }
  } else {
    int n_inner = a.n_inner, n_outer = a.n_outer;
    int64_t ostride = a.a.ostride;
    auto flat = [&](const sf_view_t& v) { return v.ostride == n_inner || n_outer == 1; };
    bool contiguous = flat(a.a) && flat(a.out) && (!a.res.ptr || flat(a.res)) &&
                      (!a.rowbias || a.rowbias_stride == 0);
    if (a.mode == SF_GEMM_PLAIN && contiguous && a.batch == 1 && (int64_t)n_inner * n_outer < (1ll << 31)) {
      n_inner = n_inner * n_outer;  // collapse to one row range
      n_outer = 1;
      ostride = n_inner;
      p.collapsed = 1;
    }
    p.n_inner = n_inner;
    // rows of a tile = bo outer x bi inner: the power-of-two split with the fewest padded
    // rows (ties -> wider bi), e.g. 144 pixels x 25 frames: 32 x 4 (80 % useful) instead
    // of 128 x 1 (56 %)
    {
      const int64_t outer = a.mode == SF_GEMM_TCONV3 ? a.T : n_outer;
      int64_t best = -1;
      for (int bi = BM; bi >= 8; bi >>= 1) {
        const int bo = BM / bi;
        const int64_t padded = (int64_t)((n_inner + bi - 1) / bi) * bi * ((outer + bo - 1) / bo) * bo;
        if (best < 0 || padded < best) {
          best = padded;
          p.bi = bi;
        }
      }
      p.bo = BM / p.bi;
    }
    p.tiles_i = (n_inner + p.bi - 1) / p.bi;
    uint64_t dims[4], str[3];
    dims[0] = (uint64_t)a.cin * p.taps / p.taps;  // channels of one tap
    dims[1] = (uint64_t)n_inner;
    str[0] = ld * es;
    str[1] = (uint64_t)(ostride ? ostride : n_inner) * ld * es;
    if (a.mode == SF_GEMM_TCONV3) {
      p.T = a.T;
      p.n_outer = a.n_outer;
      p.n_z = a.n_outer / a.T;
      p.tiles_o = (a.T + p.bo - 1) / p.bo;
      dims[2] = (uint64_t)a.T;
      dims[3] = (uint64_t)p.n_z;
      str[2] = (uint64_t)a.T * str[1];
    } else {
      p.n_outer = n_outer;
      p.n_z = a.batch;
      p.tiles_o = (n_outer + p.bo - 1) / p.bo;
      p.a_batched = a.batch > 1 && a.a_bstride != 0;
      dims[2] = (uint64_t)n_outer;
      dims[3] = p.a_batched ? (uint64_t)a.batch : 1;
      str[2] = p.a_batched ? (uint64_t)a.a_bstride * es : (uint64_t)n_outer * str[1];
    }
    p.tiles_m = (int64_t)p.tiles_i * p.tiles_o * p.n_z;
    uint32_t box[4] = {BK, (uint32_t)p.bi, (uint32_t)p.bo, 1};
    SF_CHECK_ARG(encode(&ma, a.a.ptr, 4, dims, str, box), SF_ERR_CUDA, "tensor map A");
  }
  pair = pair && p.tiles_m >= 2;
  // the two CTAs of a pair share one B tile: with a per-batch B (attention scores) a
  // pair must not straddle two batches, i.e. each batch needs an even tile count
  if (a.batch > 1 && a.mode == SF_GEMM_PLAIN && ((int64_t)p.tiles_i * p.tiles_o) % 2) pair = false;
  int BN = pick_bn(a.N);
  // 192/224-wide tiles only for long K: compute-bound convs gain (L1 conv K=17280 N=640: 914 -> 846 us),
  // memory-bound short-K GEMMs lose (K=320 N=640: 118 -> 131 us in the key step)
  const bool pair_in = pair;
  pair = choose_tiling(a.N, p.tiles_m, pair, !a.out_fp32 && p.taps * p.cblocks >= 12, &BN);
  // v^T projections (the weights as a shared A, M = C, batched over frames, many N tiles, short K,
  // no epilogue operands): memory bound on B with few M tiles, where 160-column tiles (the last one
  // partial: OOB B rows load as zeros, stores clip) measured faster than the model's pick:
  // L0 81.9 -> 73.1 us, L1 65.6 -> 57.6 us (profiles/README.md finding 21)
  if (!getenv("SF_GEMM_BN") && a.mode == SF_GEMM_PLAIN && a.batch > 1 && a.a_bstride == 0 && !a.bias &&
      !a.rowbias && !a.res.ptr && !a.out_fp32 && a.cin <= 640 && a.N >= 2048) {
    BN = 160;
    pair = pair_in;
  }
  p.BN = BN;
  p.tiles_n = (a.N + BN - 1) / BN;
  {
    const int taps = p.taps;
    uint64_t dims[3] = {(uint64_t)taps * a.cin, (uint64_t)a.N, (uint64_t)(a.batch > 1 ? a.batch : 1)};
    uint64_t str[2] = {(uint64_t)a.w_ld * es, (uint64_t)(a.batch > 1 ? a.w_bstride : a.w_ld * a.N) * es};
    uint32_t box[3] = {BK, (uint32_t)(pair ? BN / 2 : BN), 1};
    p.b_batched = a.batch > 1 && a.mode == SF_GEMM_PLAIN;
    SF_CHECK_ARG(encode(&mb, a.w, 3, dims, str, box), SF_ERR_CUDA, "tensor map B");
  }
  CUtensorMap mr = mb, mo = mb;
  tc::Maps M;
  M.a = ma;
  M.b = mb;
  M.at = p.tail_rows ? mat : ma;
  M.r = M.o = M.rt = M.ot = mb;
  if (!a.out_fp32) {
    SF_CHECK_ARG(encode_rows_map(&mo, a, p, a.out, a.out_bstride, BN), SF_ERR_CUDA, "tensor map out");
    if (a.res.ptr) SF_CHECK_ARG(encode_rows_map(&mr, a, p, a.res, a.res_bstride, BN), SF_ERR_CUDA, "tensor map res");
    M.o = M.ot = mo;
    M.r = M.rt = mr;
    if (p.tail_rows) {
      SF_CHECK_ARG(encode_rows_map(&M.ot, a, p, a.out, a.out_bstride, BN, true), SF_ERR_CUDA, "tensor map out tail");
      if (a.res.ptr)
        SF_CHECK_ARG(encode_rows_map(&M.rt, a, p, a.res, a.res_bstride, BN, true), SF_ERR_CUDA,
                     "tensor map res tail");
    }
    // long K: deep operand ring + one staging buffer; short K: double staging so the
    // epilogue (residual prefetch + TMA store) overlaps the next tile
    // (>= 12 K blocks measured on B200: K=1280 plain 49.5 -> 42.8 us, K=960 tconv -1.6 %; at
    // 10 blocks (K=640) double staging still wins)
#ifndef TC_LONGK_MIN
#define TC_LONGK_MIN 12
#endif
    const bool long_k = p.taps * p.cblocks >= TC_LONGK_MIN;
    if (pair) {
      if (long_k) {
        switch (BN) {
          case 256: return launch_cfg<256, 5, 1, true>(p, M, st);
          case 224: return launch_cfg<224, 5, 1, true>(p, M, st);
          case 192: return launch_cfg<192, 6, 1, true>(p, M, st);
          case 160: return launch_cfg<160, 7, 1, true>(p, M, st);
          case 128: return launch_cfg<128, 8, 1, true>(p, M, st);
          default: return launch_cfg<64, 10, 1, true>(p, M, st);
        }
      }
      switch (BN) {
        case 256: return launch_cfg<256, 3, 2, true>(p, M, st);
        case 224: return launch_cfg<224, 3, 2, true>(p, M, st);
        case 192: return launch_cfg<192, 4, 2, true>(p, M, st);
        case 160: return launch_cfg<160, 5, 2, true>(p, M, st);
        case 128: return launch_cfg<128, 6, 2, true>(p, M, st);
        default: return launch_cfg<64, 9, 2, true>(p, M, st);
      }
    }
    if (long_k) {
      switch (BN) {
        case 256: return launch_cfg<256, 3, 1>(p, M, st);
        case 160: return launch_cfg<160, 5, 1>(p, M, st);
        case 128: return launch_cfg<128, 6, 1>(p, M, st);
        default: return launch_cfg<64, 8, 1>(p, M, st);
      }
    }
    switch (BN) {
      case 256: return launch_cfg<256, 2, 2>(p, M, st);
      case 160: return launch_cfg<160, 4, 2>(p, M, st);
      case 128: return launch_cfg<128, 5, 2>(p, M, st);
      default: return launch_cfg<64, 7, 2>(p, M, st);
    }
  }
  // fp32 output: TMA-store epilogue (EPI 3) when rows / strides are 16-byte aligned and there
  // is no residual; otherwise direct stores (EPI 0)
  const bool f32_tma = !a.res.ptr && aligned16(a.out.ptr) && a.out.ld % 4 == 0 && (a.out.ostride * a.out.ld * 4) % 16 == 0 &&
                       (a.out_bstride * 4) % 16 == 0 && encode_rows_map(&M.o, a, p, a.out, a.out_bstride, BN, false, true) &&
                       (!p.tail_rows || encode_rows_map(&M.ot, a, p, a.out, a.out_bstride, BN, true, true));
  if (f32_tma) {
    if (pair) {
      switch (BN) {
        case 256: return launch_cfg<256, 5, 3, true>(p, M, st);
        case 160: return launch_cfg<160, 6, 3, true>(p, M, st);
        case 128: return launch_cfg<128, 6, 3, true>(p, M, st);
        default: return launch_cfg<64, 8, 3, true>(p, M, st);
      }
    }
    switch (BN) {
      case 256: return launch_cfg<256, 3, 3>(p, M, st);
      case 160: return launch_cfg<160, 4, 3>(p, M, st);
      case 128: return launch_cfg<128, 5, 3>(p, M, st);
      default: return launch_cfg<64, 6, 3>(p, M, st);
    }
  }
  if (pair) {
    switch (BN) {
      case 256: return launch_cfg<256, 6, 0, true>(p, M, st);
      case 160: return launch_cfg<160, 8, 0, true>(p, M, st);
      case 128: return launch_cfg<128, 8, 0, true>(p, M, st);
      default: return launch_cfg<64, 10, 0, true>(p, M, st);
    }
  }
  switch (BN) {
    case 256: return launch_cfg<256, 4, 0>(p, M, st);
    case 160: return launch_cfg<160, 5, 0>(p, M, st);
    case 128: return launch_cfg<128, 6, 0>(p, M, st);
    default: return launch_cfg<64, 8, 0>(p, M, st);
  }
}

}  // namespace sf
