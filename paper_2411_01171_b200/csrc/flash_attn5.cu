// Fused single-head spatial attention on CTA pairs (kernels.py:269-300):
//   O = softmax(Q K^T * scale) V per frame, head dim D = C in {128, 256, 320}.
//
// Two query tiles of one frame form a CTA pair (cluster of 2); the leader
// issues tcgen05.mma.cta_group::2 with M = 256 (rows 0-127 from the leader's
// Q/P, 128-255 from the peer's).  B operands are split along N, so each CTA
// stages half of every K block and half of every V^T block, fetched with 2-SM
// TMA whose completion is counted on the leader's barrier.
//
// Differences from v3 (flash_attn3.cu), all aimed at MMA issue efficiency —
// on B200 an M=256 N=64 tcgen05.mma costs ~50 issue cycles against a 32-cycle
// tensor floor, N >= 96 runs at the floor:
//  * KV blocks of BKV = 96 keys (D = 320) or 128 (D <= 256), so S = Q K^T is
//    issued as N = 96/128 MMAs and every per-block barrier/commit is amortised
//    over 1.5-2x more keys;
//  * P is written in place over the first BKV/2 columns of its own S buffer
//    (bf16x2), which is what lets O [0,D) + S[2] fit the 512 TMEM columns at
//    D = 320.  The next S into that buffer is issued after the P.V that reads
//    P, on the same in-order tcgen05 pipe, so no "S buffer free" barrier
//    remains; the only MMA-side wait on the softmax is p_full;
//  * V^T is staged in 32-key chunks with a 64-byte swizzle (a 96-key row
//    does not fit one 128-byte swizzle atom).
// Online softmax with a lazy max (O and l rescaled only when a row max grows
// by more than 2^8), ex2.approx, relaxed cross-CTA arrives.
// Warps: 0 TMA (both CTAs), 1 MMA issuer (leader only) + TMEM alloc,
//        2..5 softmax + epilogue (one query row per thread).
#include "common.cuh"

#include <cuda.h>
#include <mutex>

namespace sf {
namespace fa5 {

constexpr int BQ = 128, THREADS = 192;
constexpr int SMEM_CAP = 232448;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// K-major UMMA smem descriptors (sm_100 layout: start>>4, LBO 1, SBO, version 1, swizzle mode)
__device__ __forceinline__ uint64_t sdesc128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint64_t sdesc64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#define SF_R32(r) \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), \
      "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), \
      "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), \
      "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
#define SF_W16(r) \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), \
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
#define SF_W32(r) \
  SF_W16(r), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), \
      "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])

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
__device__ __forceinline__ void tst16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      SF_W16(r));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA rank 0 (the leader)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t a = smem_u32(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  return r;
}
// relaxed remote arrive: every TMEM access it publishes has completed (wait::ld/st + fence::before)
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA into my own smem; completion bytes land on the leader's barrier
__device__ __forceinline__ void tma3_2sm(const CUtensorMap* m, uint32_t bar_cluster, void* dst, int c0, int c1,
                                         int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(m), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// The MMA warp runs converged (all 32 lanes, warp-uniform descriptors) and every tcgen05
// instruction is issued by one elect.sync-chosen lane inside the asm: with the operands
// provably uniform ptxas keeps them in uniform registers and emits no per-MMA waterfall
// loop (issuing from a lane==0 branch cost ~13 SASS instructions per MMA).
// converged-warp producer variants (one elect.sync lane issues; whole warp calls)
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma3_2sm_e(const CUtensorMap* m, uint32_t bar_cluster, void* dst, int c0, int c1,
                                           int c2) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];\n}\n" ::"r"(smem_u32(dst)),
      "l"(m), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
// arrive on the barrier at this offset in both CTAs once the leader's MMAs complete
__device__ __forceinline__ void commit2(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
// bf16 x bf16 -> fp32, both operands K-major, M = 256 (cta_group::2)
__host__ __device__ constexpr uint32_t idesc256(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

struct Params {
  int HW, frames, n_kv, n_qt;
  float scale_log2;
  sf_view_t out;
};

template <int D>
struct Cfg {
  static constexpr int BKV = D == 320 ? 96 : 128;     // O [0,D) + S[2] [D, D+2*BKV) <= 512 TMEM columns
  static constexpr int NCH = D / 64;                   // 64-wide d chunks (128-byte swizzle atoms)
  static constexpr int NKC = BKV / 32;                 // 32-key chunks of V^T (64-byte swizzle atoms)
  static constexpr int Q_BYTES = NCH * BQ * 128;
  // ring items (per CTA): K half = NCH sub-tiles [BKV/2 keys x 64 d];
  //                       V^T half = 2 (d halves) x NKC chunks [D/4 d x 32 keys]
  static constexpr int K_SUB = (BKV / 2) * 128;
  static constexpr int V_CH = (D / 4) * 64;
  static constexpr int K_HALF = NCH * K_SUB;
  static constexpr int V_HALF = 2 * NKC * V_CH;
  static constexpr int SLOT = ((K_HALF > V_HALF ? K_HALF : V_HALF) + 1023) / 1024 * 1024;
  static constexpr int NSLOT_FIT = (SMEM_CAP - 1024 - 256 - Q_BYTES) / SLOT;
  static constexpr int NSLOT = NSLOT_FIT > 8 ? 8 : NSLOT_FIT;
  static constexpr int TOTAL = 1024 + Q_BYTES + NSLOT * SLOT + 256;
  static constexpr int S_COL = D;
  static_assert(D % 64 == 0 && D + 2 * BKV <= 512, "TMEM budget");
  static_assert(K_SUB % 1024 == 0 && V_CH % 512 == 0, "swizzle atom alignment");
  static_assert(NSLOT >= 3 && TOTAL <= SMEM_CAP, "shared memory budget");
};

template <int D>
__global__ void __launch_bounds__(THREADS, 1)
    flash5_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap mQ,
                  const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV) {
  using L = Cfg<D>;
  constexpr int BKV = L::BKV, NSLOT = L::NSLOT;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment by offsetting the shared array itself (a uintptr_t round trip loses
  // the shared address space: every C++ staging access became a generic LD/ST.E)
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = base;
  uint8_t* sRing = sQ + L::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sRing + NSLOT * L::SLOT);
  uint64_t* q_full = bars;              // leader: Q of both CTAs landed
  uint64_t* r_full = bars + 1;          // [NSLOT] leader: both halves of a ring item landed
  uint64_t* r_empty = r_full + NSLOT;   // [NSLOT] per CTA: item consumed
  uint64_t* s_full = r_empty + NSLOT;   // [2] per CTA: S of a block in buffer b complete
  uint64_t* p_full = s_full + 2;        // [2] leader: 8 softmax warps wrote P into buffer b
  uint64_t* o_done = p_full + 2;        // [2] per CTA: P.V of a block using buffer b complete
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int q0 = blockIdx.x * BQ, f = blockIdx.y;
  const int nkv = p.n_kv;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 8);
      mbar_init(&o_done[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  cluster_sync();
  fence_after();
  const uint32_t tmem = *tslot;
  // prologue (barriers, TMEM) done without touching global data: now wait for the
  // producing kernel (PDL) and let the next one be scheduled
  griddep_wait();

  if (warp == 0) {
    {   // whole warp converged, elect.sync issue
      // ---------------- TMA: my halves, completion counted on the leader ----------------
      if (leader) mbar_expect_tx_e(q_full, 2 * L::Q_BYTES);
      const uint32_t qbar = leader_addr(q_full);
      for (int c = 0; c < L::NCH; ++c) tma3_2sm_e(&mQ, qbar, sQ + c * BQ * 128, c * 64, q0, f);
      int slot = 0;
      uint32_t ph = 0;
      auto next = [&]() {
        if (++slot == NSLOT) {
          slot = 0;
          ph ^= 1;
        }
      };
      auto item = [&](int bytes_both) {
        mbar_wait(&r_empty[slot], ph ^ 1);
        if (leader) mbar_expect_tx_e(&r_full[slot], bytes_both);
        return leader_addr(&r_full[slot]);
      };
      auto load_k = [&](int j) {
        const uint32_t b = item(2 * L::K_HALF);
        for (int c = 0; c < L::NCH; ++c)
          tma3_2sm_e(&mK, b, sRing + slot * L::SLOT + c * L::K_SUB, c * 64, j * BKV + (int)rank * (BKV / 2), f);
        next();
      };
      load_k(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) load_k(j + 1);
        const uint32_t b = item(2 * L::V_HALF);
        for (int h = 0; h < 2; ++h)
          for (int kc = 0; kc < L::NKC; ++kc)
            tma3_2sm_e(&mV, b, sRing + slot * L::SLOT + (h * L::NKC + kc) * L::V_CH, j * BKV + kc * 32,
                     h * (D / 2) + (int)rank * (D / 4), f);
        next();
      }
      // drain: every slot's release (multicast commit) has landed before the CTA retires
      for (int s = 0; s < NSLOT; ++s) {
        mbar_wait(&r_empty[slot], ph ^ 1);
        next();
      }
    }
    griddep_trigger();   // all loads issued: let the next kernel's prologue start
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (leader only, whole warp converged), M = 256 ----------------
      constexpr uint32_t idS = idesc256(BKV), idO = idesc256(D / 2);
      mbar_wait(q_full, 0);
      fence_after();
      const uint64_t qd = sdesc128(smem_u32(sQ));
      int slot = 0;
      uint32_t ph = 0;
      auto next = [&]() {
        if (++slot == NSLOT) {
          slot = 0;
          ph ^= 1;
        }
      };
      // S(j) -> buffer j&1.  The previous reader of that buffer is P.V(j-2)
      // (its P), issued earlier on this in-order pipe.
      auto issue_S = [&](int j) {
        const int b = j & 1;
        mbar_wait(&r_full[slot], ph);
        fence_after();
        const uint64_t kd = sdesc128(smem_u32(sRing + slot * L::SLOT));
#pragma unroll
        for (int c = 0; c < L::NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma2_ss(tmem + L::S_COL + b * BKV, qd + (uint64_t)((c * BQ * 128 + k * 32) >> 4),
                    kd + (uint64_t)((c * L::K_SUB + k * 32) >> 4), idS, (c | k) != 0);
        commit2(&r_empty[slot]);
        next();
        commit2(&s_full[b]);
      };
      auto issue_PV = [&](int j) {
        const int b = j & 1;
        mbar_wait(&p_full[b], (j >> 1) & 1);
        mbar_wait(&r_full[slot], ph);
        fence_after();
        const uint32_t vbase = smem_u32(sRing + slot * L::SLOT);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint32_t pa = tmem + L::S_COL + b * BKV + (uint32_t)(k * 8);
          const uint32_t off = (uint32_t)((k >> 1) * L::V_CH + (k & 1) * 32);
          mma2_ts(tmem, pa, sdesc64(vbase + off), idO, (j | k) != 0);
          mma2_ts(tmem + D / 2, pa, sdesc64(vbase + L::NKC * L::V_CH + off), idO, (j | k) != 0);
        }
        commit2(&r_empty[slot]);
        next();
        commit2(&o_done[b]);
      };
      issue_S(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_S(j + 1);
        issue_PV(j);
      }
    }
  } else {
    // ---------------- softmax + epilogue (both CTAs, own 128 rows) ----------------
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float c = p.scale_log2;
    const uint32_t p_full_l = leader_addr(p_full);
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      const uint32_t sb = tmem + lane_off + L::S_COL + b * BKV;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      fence_after();
      uint32_t r[BKV];
#pragma unroll
      for (int k = 0; k < BKV / 32; ++k) tld32(sb + 32 * k, r + 32 * k);
      tld_wait();
      const int kbase = j * BKV;
      if (kbase + BKV > p.HW) {
#pragma unroll
        for (int e = 0; e < BKV; ++e)
          if (kbase + e >= p.HW) r[e] = __float_as_uint(-INFINITY);
      }
      float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
      for (int e = 0; e < BKV; e += 2) {
        m0 = fmaxf(m0, __uint_as_float(r[e]));
        m1 = fmaxf(m1, __uint_as_float(r[e + 1]));
      }
      const float mb = fmaxf(m0, m1) * c;
      bool need = false;
      float corr = 1.f;
      if (j == 0) {
        m_run = mb;
      } else if (mb > m_run + 8.f) {
        need = true;
        corr = ex2(m_run - mb);
        m_run = mb;
      }
      float ls0 = 0.f, ls1 = 0.f;
      uint32_t pk[BKV / 2];
#pragma unroll
      for (int e = 0; e < BKV / 2; ++e) {
        const float a0 = ex2(fmaf(__uint_as_float(r[2 * e]), c, -m_run));
        const float b0 = ex2(fmaf(__uint_as_float(r[2 * e + 1]), c, -m_run));
        ls0 += a0;
        ls1 += b0;
        bf162 h = __floats2bfloat162_rn(a0, b0);
        pk[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      if (__any_sync(0xffffffffu, need)) {
        // rescaling O needs every earlier P.V finished (block j-1 included)
        mbar_wait(&o_done[b ^ 1], ((j - 1) >> 1) & 1);
        fence_after();
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          tld32(tmem + lane_off + cc, o);
          tld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tst32(tmem + lane_off + cc, o);
        }
      }
      // P over the first BKV/2 columns of this S buffer (S already read above)
#pragma unroll
      for (int k = 0; k < BKV / 64; ++k) tst32(sb + 32 * k, pk + 32 * k);
      if constexpr ((BKV / 2) % 32 != 0) tst16(sb + (BKV / 64) * 32, pk + (BKV / 64) * 32);
      tst_wait();
      l_run = l_run * corr + ls0 + ls1;
      fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster(p_full_l + b * 8);
    }
    mbar_wait(&o_done[(nkv - 1) & 1], ((nkv - 1) >> 1) & 1);
    fence_after();
    const float inv = 1.f / l_run;
    const int qrow = q0 + row;
    const bool valid = qrow < p.HW;
    bf16* dst = reinterpret_cast<bf16*>(p.out.ptr) + ((int64_t)f * p.out.ostride + qrow) * p.out.ld;
#pragma unroll 1
    for (int cc = 0; cc < D; cc += 32) {
      uint32_t o[32];
      tld32(tmem + lane_off + cc, o);
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
  cluster_sync();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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
                 uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2}, str[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1}, es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(g), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int D>
static sf_status launch(Params p, sf_view_t q, sf_view_t k, const void* vt, cudaStream_t st) {
  using L = Cfg<D>;
  p.n_kv = (p.HW + L::BKV - 1) / L::BKV;
  const uint64_t es = 2;
  const uint64_t qst = (uint64_t)(q.ostride ? q.ostride : p.HW) * q.ld * es;
  CUtensorMap mq, mk, mv;
  SF_CHECK_ARG(enc3(&mq, q.ptr, D, p.HW, p.frames, q.ld * es, qst, 64, BQ, CU_TENSOR_MAP_SWIZZLE_128B), SF_ERR_CUDA,
               "tensor map Q");
  SF_CHECK_ARG(enc3(&mk, k.ptr, D, p.HW, p.frames, k.ld * es, qst, 64, L::BKV / 2, CU_TENSOR_MAP_SWIZZLE_128B),
               SF_ERR_CUDA, "tensor map K");
  SF_CHECK_ARG(enc3(&mv, vt, p.HW, D, p.frames, (uint64_t)p.HW * es, (uint64_t)D * p.HW * es, 32, D / 4,
                    CU_TENSOR_MAP_SWIZZLE_64B),
               SF_ERR_CUDA, "tensor map V");
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(flash5_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    init = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)((p.n_qt + 1) / 2 * 2), (unsigned)p.frames, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = L::TOTAL;
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
  cudaLaunchKernelEx(&cfg, flash5_kernel<D>, p, mq, mk, mv);
  return launch_status("sf_spatial_attention_core(v5, 2-CTA)");
}

}  // namespace fa5

bool flash5_supported(int C) { return C == 320 || C == 256 || C == 128; }

sf_status flash5_launch(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int frames, int HW, int C,
                        float scale, cudaStream_t st) {
  fa5::Params p{};
  p.HW = HW;
  p.frames = frames;
  p.n_qt = (HW + fa5::BQ - 1) / fa5::BQ;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  switch (C) {
    case 320: return fa5::launch<320>(p, q, k, vt, st);
    case 256: return fa5::launch<256>(p, q, k, vt, st);
    default: return fa5::launch<128>(p, q, k, vt, st);
  }
}

}  // namespace sf
