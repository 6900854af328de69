// Fused temporal attention on tcgen05 (kernels.py:276-308: the tokens of one pixel are its T
// frames):  out = softmax((x Wq)(x Wk)^T / sqrt(C)) (x Wv) Wo  [+ residual]
//
// One persistent CTA per SM walks 128-row tiles of bi = floor(128 / T) pixels x T frames
// (a 4-D TMA box {64 ch, bi pixels, T frames, 1}: tile row r = frame * bi + pixel) and keeps
// everything between the tile's input x and its output on chip:
//   A = x Mqk                  Mqk = Wq Wk^T log2(e) / sqrt(C)   (per layer, bf16)
//   S = A x^T                  128 x 128; a query row attends only to the rows of its own
//                              pixel (block-diagonal mask), exp2 softmax, normalised P
//   B = P x                    x read as an MN-major operand (no V^T pass)
//   Y = B Mvo (+ res)          Mvo = Wv Wo                        (per layer, bf16)
// i.e. the reference's four projections and two attention products regrouped by
// associativity, (x Wq)(x Wk)^T = (x Wq Wk^T) x^T and P (x Wv) Wo = (P x)(Wv Wo): no q/k/v
// tensor and no attention context reaches HBM (the unfused path writes and re-reads a
// 3C-wide qkv and a C-wide context per row).
//
// A, P and B never leave TMEM: each is rounded to bf16 in place (packed pairs) and fed back as
// the TMEM-side A operand of the next MMA, so shared memory holds only the x tile and a deep
// ring of weight half-tiles (the weights stream from L2 once per tile: 4 C^2 bytes).
// TMEM columns (C <= 320):  A32 [0,C) -> A16 [C, 1.5C) -> S [0,128), P16 [0,64)
//                           -> B32 [512-C, 512) -> B16 [0, C/2) -> Y [512-C, 512)
// Roles (320 threads): warp 0 TMA, warp 1 MMA issuer + TMEM owner, warps 2..9 two per TMEM
// lane quarter (column halves): bf16 packing of A and B, softmax (warps 2..5, one row per
// thread), epilogue with the residual prefetched while the last MMA runs.
#include "common.cuh"

#include <cuda.h>
#include <cstdlib>
#include <mutex>

namespace sf {
namespace ta {

constexpr int THREADS = 320, ROWS = 128, CHUNK = ROWS * 128;   // one 64-channel chunk of a tile
constexpr int SMEM_CAP = 232448;

template <int NCH>
struct Cfg {
  static constexpr int C = NCH * 64;
  static constexpr int HALF = C / 2;                   // weight stage: [C/2 output ch][64 input ch]
  static constexpr int W_STAGE = HALF * 128;
  static constexpr int NW_FIT = (SMEM_CAP - 1024 - 1536 - NCH * CHUNK) / W_STAGE;
  static constexpr int NW = NW_FIT > 12 ? 12 : NW_FIT; // weight ring slots
  static constexpr int X_OFF = 0, W_OFF = NCH * CHUNK;
  static constexpr int BAR_OFF = W_OFF + NW * W_STAGE;
  static constexpr int BAR_BYTES = (2 + 2 * NW + 14) * 8 + 8;  // mbarriers + TMEM slot
  static constexpr int INV_OFF = BAR_OFF + 512;                // float[2][128]: softmax row max / sum
  static constexpr int TOTAL = 1024 + INV_OFF + 1024;
  // TMEM column map (see the header)
  static constexpr int A32 = 0, A16 = C, S = 0, B32 = 512 - C, B16 = 0, Y = 512 - C;
  // B = P x in two N pieces split on a 64-channel (swizzle atom) boundary: [0, NLO), [NLO, C)
  static constexpr int NLO = HALF / 64 * 64;
  static_assert(NLO >= 64 && C - NLO <= 256, "B pieces");
  static_assert(C >= 128 && C + C / 2 <= 512 && 128 <= 512 - C, "TMEM column map");
  static_assert(W_STAGE % 1024 == 0, "swizzle atom alignment");
  static_assert(NW >= 3 && BAR_BYTES <= 512 && TOTAL <= SMEM_CAP, "shared memory budget");
};
struct Params {
  int T, bi, R;            // frames per pixel, pixels per tile, used rows per tile (bi * T)
  int n_inner, n_pg;       // pixels per frame (band), pixel groups per batch
  int64_t n_tiles;
  sf_view_t res, out;      // rows (b*T + t, pixel)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
// converged-warp producers: one elect.sync lane issues
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma4_e(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2, int c3) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void tma2_e(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n}\n" ::
          "r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// K-major SWIZZLE_128B operand: 8-row x 128-byte atoms, SBO = 1024 B (LBO unused)
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// MN-major SWIZZLE_128B operand (the x tile read as [k = key row][n = channel]): in 16-byte
// units ((8, n), (8, k)) : ((1, LBO), (8, SBO)) -- 64 channels contiguous in a 128-byte row,
// 64-channel blocks LBO = one tile chunk apart, 8-row groups SBO = 1024 B apart
__device__ __forceinline__ uint64_t mndesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(CHUNK >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16: D fp32, A/B bf16, M = 128; b_mn: B operand MN-major
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn = false) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (b_mn ? (1u << 16) : 0u) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

#define TA_R32(r) \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
      "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), \
      "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), \
      "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define TA_W32(r) \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), \
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), \
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), \
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])

__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : TA_R32(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      TA_W32(r));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void tst16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ uint32_t pack2(uint32_t a, uint32_t b) {
  bf162 h = __floats2bfloat162_rn(__uint_as_float(a), __uint_as_float(b));
  return *reinterpret_cast<uint32_t*>(&h);
}

// n fp32 accumulator columns at src -> n/2 packed bf16 pairs at dst (the row's TMEM-side MMA
// operand); src and dst ranges are disjoint
template <int N>
__device__ __forceinline__ void pack_cols(uint32_t src, uint32_t dst) {
#pragma unroll 1
  for (int c = 0; c < N; c += 32) {
    uint32_t v[32], pk[16];
    tld32(src + c, v);
    tld_wait();
#pragma unroll
    for (int e = 0; e < 16; ++e) pk[e] = pack2(v[2 * e], v[2 * e + 1]);
    tst16(dst + c / 2, pk);
  }
  tst_wait();
}

// -DTA_TRACE (tuning builds only): SM-clock stamps of CTA 0's pipeline events per role
// (0 MMA warp, 1 warp 2 = half 0, 2 warp 6 = half 1); read with sf_debug_ta_trace
#ifdef TA_TRACE
__device__ unsigned long long g_ta_trace[3][1024];
__device__ unsigned int g_ta_n[3];
#define TA_TR(role, code)                                                                       \
  do {                                                                                          \
    if (blockIdx.x == 0 && lane == 0) {                                                         \
      const unsigned i_ = g_ta_n[role]++;                                                       \
      if (i_ < 1024) g_ta_trace[role][i_] = ((unsigned long long)clock64() << 8) | (code);      \
    }                                                                                           \
  } while (0)
#else
#define TA_TR(role, code) \
  do {                    \
  } while (0)
#endif

template <int NCH>
__global__ void __launch_bounds__(THREADS, 1)
    tattn_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap mX,
                 const __grid_constant__ CUtensorMap mW) {
  using L = Cfg<NCH>;
  constexpr int C = L::C, HALF = L::HALF, NW = L::NW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = base + L::X_OFF;
  uint8_t* sW = base + L::W_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  uint64_t* x_full = bars;          // TMA: x tile landed
  uint64_t* x_empty = bars + 1;     // MMA: last read of the x tile (B = P x) done
  uint64_t* w_full = bars + 2;      // [NW]
  uint64_t* w_empty = w_full + NW;  // [NW]
  uint64_t* a_full = w_empty + NW;  // [2] MMA: column half h of A = x Mqk in TMEM
  uint64_t* a_st = a_full + 2;      // [2] 4 warps of half h: A half packed to bf16
  uint64_t* s_full = a_st + 2;      // MMA: S in TMEM
  uint64_t* p_full = s_full + 1;    // 8 warps: P written over S
  uint64_t* b_full = p_full + 1;    // [2] MMA: B = P x columns of half h in TMEM
  uint64_t* b_st = b_full + 2;      // [2] 4 warps of half h: B half packed
  uint64_t* y_full = b_st + 2;      // [2] MMA: output half h of Y in TMEM
  uint64_t* y_free = y_full + 2;    // [2] 4 warps of half h: Y half read out of TMEM
  uint32_t* tslot = reinterpret_cast<uint32_t*>(y_free + 2);
  float* red = reinterpret_cast<float*>(base + L::INV_OFF);   // [2 halves][128 rows] row max / sum

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(x_full, 1);
    mbar_init(x_empty, 1);
    for (int s = 0; s < NW; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&a_full[h], 1);
      mbar_init(&a_st[h], 4);
      mbar_init(&b_full[h], 1);
      mbar_init(&b_st[h], 4);
      mbar_init(&y_full[h], 1);
      mbar_init(&y_free[h], 4);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rows R..127 of the x tile are never written by TMA (the box has R rows): zero them once, so
  // the padded keys / queries contribute exact zeros
  for (int idx = threadIdx.x; idx < NCH * (ROWS - p.R) * 8; idx += THREADS) {
    const int j = idx / ((ROWS - p.R) * 8), rem = idx % ((ROWS - p.R) * 8);
    *reinterpret_cast<uint4*>(sX + j * CHUNK + (p.R + rem / 8) * 128 + (rem % 8) * 16) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  griddep_wait();

  const int64_t t0 = blockIdx.x, dt = gridDim.x;
  if (warp == 0) {
    // ---------------- TMA producer ----------------
    int slot = 0;
    uint32_t wph = 0;
    auto wload = [&](int k0, int n0) {
      mbar_wait(&w_empty[slot], wph ^ 1);
      mbar_expect_tx_e(&w_full[slot], L::W_STAGE);
      tma2_e(&mW, &w_full[slot], sW + slot * L::W_STAGE, k0, n0);
      if (++slot == NW) {
        slot = 0;
        wph ^= 1;
      }
    };
    uint32_t it = 0;
    for (int64_t t = t0; t < p.n_tiles; t += dt, ++it) {
      const int z = (int)(t / p.n_pg), i0 = (int)(t % p.n_pg) * p.bi;
      mbar_wait(x_empty, (it & 1) ^ 1);
      mbar_expect_tx_e(x_full, NCH * 128 * p.R);
      for (int j = 0; j < NCH; ++j) tma4_e(&mX, x_full, sX + j * CHUNK, j * 64, i0, 0, z);
      for (int h = 0; h < 2; ++h)
        for (int j = 0; j < NCH; ++j) wload(j * 64, h * HALF);        // Mqk^T, output half h
      for (int h = 0; h < 2; ++h)
        for (int j = 0; j < NCH; ++j) wload(j * 64, C + h * HALF);    // Mvo^T, output half h
    }
    // drain: every weight slot released before the CTA retires
    for (int s = 0; s < NW; ++s) {
      mbar_wait(&w_empty[slot], wph ^ 1);
      if (++slot == NW) {
        slot = 0;
        wph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int slot = 0;
    uint32_t wph = 0;
    const uint32_t xb = smem_u32(sX), wb = smem_u32(sW);
    // output half h of D (at dcol) = A x W^T over NCH weight stages; A from the x tile (smem)
    // or, a_tmem >= 0, packed bf16 in TMEM
    auto gemm_half = [&](uint32_t dcol, int a_tmem, int h) {
#pragma unroll 1
      for (int j = 0; j < NCH; ++j) {
        mbar_wait(&w_full[slot], wph);
        fence_after();
        const uint64_t bd = kdesc(wb + slot * L::W_STAGE);
        const uint32_t d = tmem + dcol + h * HALF;
        if (a_tmem < 0) {
          const uint64_t ad = kdesc(xb + j * CHUNK);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ss(d, ad + 2 * k, bd + 2 * k, idesc(HALF), (j | k) != 0);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ts(d, tmem + a_tmem + (j * 4 + k) * 8, bd + 2 * k, idesc(HALF), (j | k) != 0);
        }
        commit_e(&w_empty[slot]);
        if (++slot == NW) {
          slot = 0;
          wph ^= 1;
        }
      }
    };
    uint32_t it = 0;
    for (int64_t t = t0; t < p.n_tiles; t += dt, ++it) {
      const uint32_t ph = it & 1;
      mbar_wait(x_full, ph);
      TA_TR(0, 1);
      fence_after();
      // A = x Mqk.  Half 0 ([0, C/2)) overlaps only operands the in-order pipe has consumed,
      // so it runs under the previous tile's epilogue; half 1 overlaps that tile's Y half 0
      gemm_half(L::A32, -1, 0);
      commit_e(&a_full[0]);
      TA_TR(0, 2);
      mbar_wait(&y_free[0], ph ^ 1);
      TA_TR(0, 3);
      fence_after();
      gemm_half(L::A32, -1, 1);
      commit_e(&a_full[1]);
      TA_TR(0, 4);
      mbar_wait(&a_st[0], ph);
      mbar_wait(&a_st[1], ph);
      TA_TR(0, 5);
      fence_after();
#pragma unroll 1
      for (int j = 0; j < NCH; ++j) {   // S = A x^T (x rows as the K-major B: [n = key][k = ch])
        const uint64_t bd = kdesc(xb + j * CHUNK);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_ts(tmem + L::S, tmem + L::A16 + (j * 4 + k) * 8, bd + 2 * k, idesc(128), (j | k) != 0);
      }
      commit_e(s_full);
      TA_TR(0, 6);
      mbar_wait(p_full, ph);
      TA_TR(0, 7);
      fence_after();
      // B = P x: 16 keys per step, x MN-major, in two N pieces on swizzle-atom boundaries.
      // The high piece [NLO, C) holds all of column half 1 and goes first: half 1 is packed
      // into B16 [C/4, C/2) while the low piece still reads P -- disjoint from P [0, 64) when
      // C >= 256; half 0's B16 [0, C/4) overlaps P, so it waits for the whole product
#pragma unroll
      for (int k = 0; k < 8; ++k)
        mma_ts(tmem + L::B32 + L::NLO, tmem + L::S + k * 8, mndesc(xb + (L::NLO / 64) * CHUNK + k * 2048),
               idesc(C - L::NLO, true), k != 0);
      if (C >= 256) commit_e(&b_full[1]);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        mma_ts(tmem + L::B32, tmem + L::S + k * 8, mndesc(xb + k * 2048), idesc(L::NLO, true), k != 0);
      commit_e(x_empty);
      commit_e(&b_full[0]);
      if (C < 256) commit_e(&b_full[1]);
      TA_TR(0, 9);
      mbar_wait(&b_st[0], ph);
      mbar_wait(&b_st[1], ph);
      TA_TR(0, 10);
      fence_after();
      gemm_half(L::Y, L::B16, 0);   // Y = B Mvo, output half 0 ...
      commit_e(&y_full[0]);
      TA_TR(0, 11);
      gemm_half(L::Y, L::B16, 1);   // ... and half 1
      commit_e(&y_full[1]);
      TA_TR(0, 12);
    }
  } else {
    // ---------------- packing / softmax / epilogue: tile row r, column half g ----------------
    const int g = (warp - 2) >> 2;
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int pix = r % p.bi, fr = r / p.bi;
    const bool live = r < p.R;
    uint32_t kmask[2];   // my keys among [64 g, 64 g + 64): pix + k * bi, k < T
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      kmask[w] = 0u;
      for (int e = 0; e < 32; ++e) {
        const int c = 64 * g + 32 * w + e;
        if (live && c < p.R && c % p.bi == pix) kmask[w] |= 1u << e;
      }
    }
    uint32_t it = 0;
    for (int64_t t = t0; t < p.n_tiles; t += dt, ++it) {
      const uint32_t ph = it & 1;
      const int z = (int)(t / p.n_pg), i0 = (int)(t % p.n_pg) * p.bi;
      // my half of A -> bf16 operand
      const int role = (warp == 2) ? 1 : (warp == 6) ? 2 : -1;
#define TA_TRW(code) do { if (role > 0) TA_TR(role, code); } while (0)
      mbar_wait(&a_full[g], ph);
      TA_TRW(20);
      fence_after();
      pack_cols<HALF>(trow + L::A32 + g * HALF, trow + L::A16 + g * (HALF / 2));
      TA_TRW(21);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_st[g]);
      // softmax over this row's keys (same pixel, frames 0..T-1); each half of the CTA holds 64
      // keys of the row: row max exchanged through shared memory, the unnormalised P packed over
      // S, 1/sum applied to Y in the epilogue (it commutes with (P x) Mvo)
      mbar_wait(s_full, ph);
      TA_TRW(22);
      fence_after();
      uint32_t sv[64];
      tld32(trow + L::S + 64 * g, sv);
      tld32(trow + L::S + 64 * g + 32, sv + 32);
      tld_wait();
      float m = -INFINITY;
#pragma unroll
      for (int e = 0; e < 64; ++e)
        if ((kmask[e >> 5] >> (e & 31)) & 1u) m = fmaxf(m, __uint_as_float(sv[e]));
      red[g * 128 + r] = m;
      asm volatile("bar.sync 1, 256;" ::: "memory");   // both halves' S read, maxima published
      TA_TRW(23);
      m = fmaxf(m, red[(g ^ 1) * 128 + r]);
      float sum = 0.f;
      uint32_t pk[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float a0 = ((kmask[(2 * e) >> 5] >> ((2 * e) & 31)) & 1u) ? ex2(__uint_as_float(sv[2 * e]) - m) : 0.f;
        const float a1 =
            ((kmask[(2 * e + 1) >> 5] >> ((2 * e + 1) & 31)) & 1u) ? ex2(__uint_as_float(sv[2 * e + 1]) - m) : 0.f;
        sum += a0 + a1;
        pk[e] = pack2(__float_as_uint(a0), __float_as_uint(a1));
      }
      tst32(trow + L::S + 32 * g, pk);
      tst_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      TA_TRW(24);
      asm volatile("bar.sync 1, 256;" ::: "memory");   // maxima consumed before the sums reuse red
      red[g * 128 + r] = sum;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const float inv = live ? 1.f / (sum + red[(g ^ 1) * 128 + r]) : 0.f;
      TA_TRW(25);
      // my half of B -> bf16 operand
      mbar_wait(&b_full[g], ph);
      TA_TRW(26);
      fence_after();
      pack_cols<HALF>(trow + L::B32 + g * HALF, trow + L::B16 + g * (HALF / 2));
      TA_TRW(27);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&b_st[g]);
      // epilogue, output half g: residual prefetched while Y = B Mvo runs, then Y/sum (+ res)
      const int i = i0 + pix;
      const bool valid = live && i < p.n_inner;
      const int64_t o = (int64_t)z * p.T + fr;
      bf16* dst = valid ? row_ptr<bf16>(p.out, o, i) + g * HALF : nullptr;
      // residual: the first two 32-column chunks prefetched while Y = B Mvo runs, then two
      // chunks ahead (a whole half row in registers spilled the packing loops)
      constexpr int NCC = HALF / 32;
      uint4 rr[2][4];
      const bool has_res = valid && p.res.ptr;
      const uint4* rs = has_res ? reinterpret_cast<const uint4*>(row_ptr<const bf16>(p.res, o, i) + g * HALF) : nullptr;
#pragma unroll
      for (int c = 0; c < 2 && c < NCC; ++c)
#pragma unroll
        for (int u = 0; u < 4; ++u) rr[c][u] = has_res ? __ldg(rs + 4 * c + u) : make_uint4(0, 0, 0, 0);
      TA_TRW(28);
      mbar_wait(&y_full[g], ph);
      TA_TRW(29);
      fence_after();
#pragma unroll
      for (int c = 0; c < NCC; ++c) {
        uint32_t y[32];
        tld32(trow + L::Y + g * HALF + 32 * c, y);
        tld_wait();
        if (valid) {
          float v[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(y[e]) * inv;
          if (has_res) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float f[8];
              unpack8(*reinterpret_cast<const bf16x8*>(&rr[c & 1][u]), f);
#pragma unroll
              for (int e = 0; e < 8; ++e) v[8 * u + e] += f[e];
            }
            if (c + 2 < NCC) {
#pragma unroll
              for (int u = 0; u < 4; ++u) rr[c & 1][u] = __ldg(rs + 4 * (c + 2) + u);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) reinterpret_cast<bf16x8*>(dst + 32 * c)[u] = pack8(v + 8 * u);
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&y_free[g]);
      TA_TRW(30);
      // both halves done with this tile's Y and sums before either packs the next tile's A
      // into columns that overlap the other half's Y
      asm volatile("bar.sync 1, 256;" ::: "memory");
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
static bool encode(CUtensorMap* m, const void* g, int rank, const uint64_t* dims, const uint64_t* strides,
                   const uint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t d[4], s[3];
  cuuint32_t b[4], es[4] = {1, 1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    if (i + 1 < rank) s[i] = strides[i];
  }
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(g), d, s, b, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NCH>
static sf_status launch(const Params& p, const sf_view_t& x, const void* w, cudaStream_t st) {
  using L = Cfg<NCH>;
  constexpr int C = L::C;
  const uint64_t es = 2, ost = (uint64_t)(x.ostride ? x.ostride : p.n_inner);
  CUtensorMap mx, mw;
  {
    const uint64_t nb = (uint64_t)p.n_tiles / p.n_pg;   // batches
    uint64_t dims[4] = {(uint64_t)C, (uint64_t)p.n_inner, (uint64_t)p.T, nb};
    uint64_t str[3] = {(uint64_t)x.ld * es, ost * x.ld * es, (uint64_t)p.T * ost * x.ld * es};
    uint32_t box[4] = {64, (uint32_t)p.bi, (uint32_t)p.T, 1};
    SF_CHECK_ARG(encode(&mx, x.ptr, 4, dims, str, box), SF_ERR_CUDA, "tensor map x (temporal attention)");
  }
  {
    uint64_t dims[2] = {(uint64_t)C, (uint64_t)(2 * C)};
    uint64_t str[1] = {(uint64_t)C * es};
    uint32_t box[2] = {64, (uint32_t)L::HALF};
    SF_CHECK_ARG(encode(&mw, w, 2, dims, str, box), SF_ERR_CUDA, "tensor map weights (temporal attention)");
  }
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(tattn_kernel<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    init = true;
  }
  const int64_t grid = p.n_tiles < num_sms() ? p.n_tiles : num_sms();
  launch_k(tattn_kernel<NCH>, dim3((unsigned)grid), dim3(THREADS), L::TOTAL, st, p, mx, mw);
  return launch_status("sf_temporal_attention_fused");
}

}  // namespace ta

// ---------------------------------------------------------------------------------------------
// Temporal attention CORE on tcgen05 for long clips (32 < T <= 128: BASELINE C4's T = 64 at the
// C >= 640 levels, where the fused kernel's x tile and accumulator do not fit): q | k | v rows
// already projected (the QKV GEMM), out = softmax(q k^T * scale) v per pixel over its T frames.
// Same tiles as the fused kernel (bi = floor(128 / T) pixels x T frames per 128 rows, block-
// diagonal mask), HBM-bound: q, k and v stream through a ring of 64-channel chunks (4-D TMA
// boxes of the qkv view), S = sum_c Q_c K_c^T accumulates in TMEM [0, 128), the unnormalised P is
// packed over S, and O = P V_j is produced one 64-channel chunk at a time (V read MN-major) into a
// 4-deep ring of TMEM buffers that the epilogue warps drain (1/rowsum applied there) while the
// next chunks multiply.  Warps: 0 TMA, 1 MMA, 2..5 softmax, 6..9 epilogue (one tile row each).
// ---------------------------------------------------------------------------------------------
namespace tcore {

constexpr int THREADS = 320, CHUNK = 128 * 128, NSLOT = 12, NOB = 4;
constexpr int SLOT_OFF = 0, BAR_OFF = NSLOT * CHUNK, INV_OFF = BAR_OFF + 512;
constexpr int TOTAL = 1024 + INV_OFF + 1024;
static_assert(TOTAL <= ta::SMEM_CAP, "shared memory budget");

struct Params {
  int T, bi, R, n_inner, n_pg, nch, koff, voff;
  int64_t n_tiles;
  float scale_log2;
  sf_view_t out;
};

__global__ void __launch_bounds__(THREADS, 1) tcore_kernel(const __grid_constant__ Params p,
                                                           const __grid_constant__ CUtensorMap mQKV) {
  using namespace ta;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* ring = base + SLOT_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + BAR_OFF);
  uint64_t* r_full = bars;                // [NSLOT]
  uint64_t* r_empty = r_full + NSLOT;     // [NSLOT]
  uint64_t* s_full = r_empty + NSLOT;     // MMA: S of the tile in TMEM
  uint64_t* p_full = s_full + 1;          // 4 softmax warps: P packed over S
  uint64_t* o_full = p_full + 1;          // [NOB] MMA: O chunk in buffer b
  uint64_t* o_free = o_full + NOB;        // [NOB] 4 epilogue warps: buffer b read
  uint64_t* inv_ready = o_free + NOB;     // [2] softmax: 1/rowsum of the tile (parity) written
  uint64_t* inv_free = inv_ready + 2;     // [2] epilogue: ... read
  uint32_t* tslot = reinterpret_cast<uint32_t*>(inv_free + 2);
  float* inv_sum = reinterpret_cast<float*>(base + INV_OFF);   // [2][128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    for (int b = 0; b < NOB; ++b) {
      mbar_init(&o_full[b], 1);
      mbar_init(&o_free[b], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&inv_ready[b], 4);
      mbar_init(&inv_free[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // rows R..127 of every ring slot stay zero (the TMA box has R rows)
  for (int idx = threadIdx.x; idx < NSLOT * (128 - p.R) * 8; idx += THREADS) {
    const int j = idx / ((128 - p.R) * 8), rem = idx % ((128 - p.R) * 8);
    *reinterpret_cast<uint4*>(ring + j * CHUNK + (p.R + rem / 8) * 128 + (rem % 8) * 16) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  griddep_wait();

  const int64_t t0 = blockIdx.x, dt = gridDim.x;
  const int nch = p.nch;
  if (warp == 0) {
    // ---------------- TMA: Q_0 K_0 Q_1 K_1 ... then V_0 V_1 ... per tile ----------------
    int slot = 0;
    uint32_t ph = 0;
    auto load = [&](int col, int i0, int z) {
      mbar_wait(&r_empty[slot], ph ^ 1);
      mbar_expect_tx_e(&r_full[slot], 128 * p.R);
      tma4_e(&mQKV, &r_full[slot], ring + slot * CHUNK, col, i0, 0, z);
      if (++slot == NSLOT) {
        slot = 0;
        ph ^= 1;
      }
    };
    for (int64_t t = t0; t < p.n_tiles; t += dt) {
      const int z = (int)(t / p.n_pg), i0 = (int)(t % p.n_pg) * p.bi;
      for (int c = 0; c < nch; ++c) {
        load(c * 64, i0, z);
        load(p.koff + c * 64, i0, z);
      }
      for (int c = 0; c < nch; ++c) load(p.voff + c * 64, i0, z);
    }
    for (int s = 0; s < NSLOT; ++s) {   // drain: every slot released before the CTA retires
      mbar_wait(&r_empty[slot], ph ^ 1);
      if (++slot == NSLOT) {
        slot = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int slot = 0;
    uint32_t ph = 0;
    int ob = 0;
    uint32_t oph = 0;
    const uint32_t rb = smem_u32(ring);
    auto next = [&]() {
      if (++slot == NSLOT) {
        slot = 0;
        ph ^= 1;
      }
    };
    uint32_t it = 0;
    for (int64_t t = t0; t < p.n_tiles; t += dt, ++it) {
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {     // S += Q_c K_c^T
        const int sq = slot;
        mbar_wait(&r_full[sq], ph);
        next();
        const int sk = slot;
        mbar_wait(&r_full[sk], ph);
        fence_after();
        const uint64_t ad = kdesc(rb + sq * CHUNK), bd = kdesc(rb + sk * CHUNK);
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_ss(tmem, ad + 2 * k, bd + 2 * k, idesc(128), (c | k) != 0);
        commit_e(&r_empty[sq]);
        commit_e(&r_empty[sk]);
        next();
      }
      commit_e(s_full);
      mbar_wait(p_full, it & 1);
      fence_after();
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {     // O_c = P V_c into TMEM buffer ob
        mbar_wait(&r_full[slot], ph);
        mbar_wait(&o_free[ob], oph ^ 1);
        fence_after();
        const uint32_t vb = rb + slot * CHUNK;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          mma_ts(tmem + 128 + ob * 64, tmem + k * 8, mndesc(vb + k * 2048), idesc(64, true), k != 0);
        commit_e(&r_empty[slot]);
        commit_e(&o_full[ob]);
        next();
        if (++ob == NOB) {
          ob = 0;
          oph ^= 1;
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- softmax (one tile row per thread) ----------------
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int pix = r % p.bi;
    const bool live = r < p.R;
    uint32_t kmask[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      kmask[w] = 0u;
      for (int e = 0; e < 32; ++e) {
        const int c = 32 * w + e;
        if (live && c < p.R && c % p.bi == pix) kmask[w] |= 1u << e;
      }
    }
    const float sl = p.scale_log2;
    uint32_t it = 0;
    for (int64_t t = t0; t < p.n_tiles; t += dt, ++it) {
      mbar_wait(s_full, it & 1);
      fence_after();
      float m = -INFINITY;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t sv[32];
        tld32(trow + 32 * k, sv);
        tld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if ((kmask[k] >> e) & 1u) m = fmaxf(m, __uint_as_float(sv[e]));
      }
      m *= sl;
      float sum = 0.f;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t sv[32], pk[16];
        tld32(trow + 32 * k, sv);
        tld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float x = ((kmask[k] >> e) & 1u) ? ex2(fmaf(__uint_as_float(sv[e]), sl, -m)) : 0.f;
          sv[e] = __float_as_uint(x);
          sum += x;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack2(sv[2 * e], sv[2 * e + 1]);
        tst16(trow + 16 * k, pk);   // packed chunk k lands on columns already read
      }
      tst_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      const int ib = it & 1;
      mbar_wait(&inv_free[ib], ((it >> 1) & 1) ^ 1);
      inv_sum[ib * 128 + r] = live ? 1.f / sum : 0.f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&inv_ready[ib]);
    }
  } else {
    // ---------------- epilogue: O chunks (1/rowsum) -> out rows ----------------
    const int q = warp & 3, r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const int pix = r % p.bi, fr = r / p.bi;
    const bool live = r < p.R;
    int ob = 0;
    uint32_t oph = 0;
    uint32_t it = 0;
    for (int64_t t = t0; t < p.n_tiles; t += dt, ++it) {
      const int z = (int)(t / p.n_pg), i0 = (int)(t % p.n_pg) * p.bi;
      const int i = i0 + pix;
      const bool valid = live && i < p.n_inner;
      bf16* dst = valid ? row_ptr<bf16>(p.out, (int64_t)z * p.T + fr, i) : nullptr;
      const int ib = it & 1;
      mbar_wait(&inv_ready[ib], (it >> 1) & 1);
      const float inv = inv_sum[ib * 128 + r];
      __syncwarp();
      if (lane == 0) mbar_arrive(&inv_free[ib]);
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&o_full[ob], oph);
        fence_after();
        uint32_t a[32], b2[32];
        tld32(trow + 128 + ob * 64, a);
        tld32(trow + 128 + ob * 64 + 32, b2);
        tld_wait();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[ob]);
        if (valid) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(a[8 * u + e]) * inv;
            reinterpret_cast<bf16x8*>(dst + c * 64)[u] = pack8(v);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(b2[8 * u + e]) * inv;
            reinterpret_cast<bf16x8*>(dst + c * 64)[4 + u] = pack8(v);
          }
        }
        if (++ob == NOB) {
          ob = 0;
          oph ^= 1;
        }
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

}  // namespace tcore


// internal entry points of sf_temporal_attention_core (elementwise.cu); C linkage, not in the header
extern "C" __attribute__((visibility("hidden"))) bool temporal_core_tc_supported(int T, int C, int koff, int voff, sf_view_t qkv, sf_view_t out) {
  static const int min_t = getenv("SF_TCORE_MIN_T") ? atoi(getenv("SF_TCORE_MIN_T")) : 33;   // A/B knob
  return T >= min_t && T <= 128 && C % 64 == 0 && koff % 64 == 0 && voff % 64 == 0 && aligned16(qkv.ptr) &&
         qkv.ld % 8 == 0 && view_vec8_ok(out);
}

extern "C" __attribute__((visibility("hidden"))) sf_status temporal_core_tc_launch(
    sf_view_t qkv, int koff, int voff, sf_view_t out, int B, int T, int n_inner, int C, float scale, cudaStream_t st) {
  tcore::Params p{};
  p.T = T;
  p.bi = 128 / T;
  p.R = p.bi * T;
  p.n_inner = n_inner;
  p.n_pg = (n_inner + p.bi - 1) / p.bi;
  p.n_tiles = (int64_t)B * p.n_pg;
  p.nch = C / 64;
  p.koff = koff;
  p.voff = voff;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  const uint64_t es = 2, ost = (uint64_t)(qkv.ostride ? qkv.ostride : n_inner);
  CUtensorMap m;
  uint64_t dims[4] = {(uint64_t)(voff + C), (uint64_t)n_inner, (uint64_t)T, (uint64_t)B};
  uint64_t str[3] = {(uint64_t)qkv.ld * es, ost * qkv.ld * es, (uint64_t)T * ost * qkv.ld * es};
  uint32_t box[4] = {64, (uint32_t)p.bi, (uint32_t)T, 1};
  SF_CHECK_ARG(ta::encode(&m, qkv.ptr, 4, dims, str, box), SF_ERR_CUDA, "tensor map qkv (temporal core)");
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(tcore::tcore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tcore::TOTAL);
    init = true;
  }
  const int64_t grid = p.n_tiles < num_sms() ? p.n_tiles : num_sms();
  launch_k(tcore::tcore_kernel, dim3((unsigned)grid), dim3(tcore::THREADS), tcore::TOTAL, st, p, m);
  return launch_status("sf_temporal_attention_core(tcgen05)");
}

#ifdef TA_TRACE
extern "C" int32_t sf_debug_ta_trace(unsigned long long* host, uint32_t* counts) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(counts, ta::g_ta_n, sizeof(unsigned) * 3);
  cudaMemcpyFromSymbol(host, ta::g_ta_trace, sizeof(unsigned long long) * 3 * 1024);
  const unsigned zero[3] = {0, 0, 0};
  cudaMemcpyToSymbol(ta::g_ta_n, zero, sizeof(zero));
  return 0;
}
#endif

extern "C" int32_t sf_temporal_attention_fused_supported(int32_t T, int32_t C) {
  return T >= 1 && T <= 128 && C >= 128 && C <= 320 && C % 64 == 0;
}

extern "C" sf_status sf_temporal_attention_fused(sf_view_t x, const void* w, sf_view_t res, sf_view_t out, int32_t B,
                                                 int32_t T, int32_t n_inner, int32_t C, void* stream) {
  SF_CHECK_ARG(sf_temporal_attention_fused_supported(T, C), SF_ERR_SHAPE, "fused temporal attention: T <= 128, C in {128, 192, 256, 320}");
  SF_CHECK_ARG(x.ptr && w && out.ptr, SF_ERR_PARAM, "null buffer");
  SF_CHECK_ARG(B >= 1 && n_inner >= 1, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(aligned16(x.ptr) && aligned16(w) && x.ld % 8 == 0 && view_vec8_ok(out) &&
                   (!res.ptr || view_vec8_ok(res)),
               SF_ERR_PARAM, "16-byte aligned rows required");
  ta::Params p{};
  p.T = T;
  p.bi = 128 / T;
  p.R = p.bi * T;
  p.n_inner = n_inner;
  p.n_pg = (n_inner + p.bi - 1) / p.bi;
  p.n_tiles = (int64_t)B * p.n_pg;
  p.res = res;
  p.out = out;
  cudaStream_t st = (cudaStream_t)stream;
  switch (C / 64) {
    case 5: return ta::launch<5>(p, x, w, st);
    case 4: return ta::launch<4>(p, x, w, st);
    case 3: return ta::launch<3>(p, x, w, st);
    default: return ta::launch<2>(p, x, w, st);
  }
}

}  // namespace sf
