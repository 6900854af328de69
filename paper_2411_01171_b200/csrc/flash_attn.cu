// Fused single-head spatial attention on tcgen05 (kernels.py:269-300):
//   O = softmax(Q K^T * scale) V,   one frame = one sequence of HW tokens,
//   head_dim D = C (the reference never splits heads), D <= 320.
//
// One CTA = 128 query rows of one frame; loop over key blocks of 64:
//   S_j = Q K_j^T            tcgen05.mma M=128 N=64,  A=Q (smem), B=K_j (smem)
//   P_j = exp2(S_j*c - m)    softmax warps: TMEM -> regs -> bf16 P in smem (SW128)
//   O  += P_j V_j            tcgen05.mma M=128 N=D/2 x2, A=P (smem), B=V^T_j (smem)
// O (D fp32 columns) and two S buffers (2 x 64 columns) live in TMEM (<= 448 of
// 512 columns).  Online softmax with a lazy max: O/l are rescaled only when a
// row's max grows by more than 2^8, so the final normalisation is exact.
// Q (D/64 SW128 chunks) is loaded once; K_j and V_j stream through a 3-slot
// TMA ring in consumption order K_0, K_1, V_0, K_2, V_1, ...  (the MMA warp
// issues S_{j+1} before P_j V_j so the softmax of block j overlaps the tensor
// core).  V is consumed as V^T [D][HW] (K-major B), produced by the projection.
//
// Warps: 0 = TMA, 1 = MMA issuer (+TMEM alloc), 2..5 = softmax + epilogue.
#include "common.cuh"

#include <cuda.h>
#include <cstdlib>
#include <mutex>

namespace sf {
namespace fa {

constexpr int BQ = 128, BKV = 64, THREADS = 192;
constexpr int SLOTS = 3;

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
__device__ __forceinline__ void tma3_mc(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                        uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

struct Params {
  int HW, frames;
  int n_kv;               // key blocks
  float scale_log2;       // (1/sqrt(D)) * log2(e)
  sf_view_t out;          // o rows: (frame, token)
};

template <int D>
struct Layout {
  static constexpr int NCH = D / 64;                  // 64-wide d chunks
  static constexpr int Q_BYTES = NCH * BQ * 128;      // NCH x [128 rows x 128 B]
  static constexpr int SLOT_BYTES = NCH * BKV * 128;  // K_j: NCH x [64 x 128 B]; V^T_j: 2 x [D/2 x 128 B]
  static constexpr int P_BYTES = BQ * 128;
  static constexpr int TOTAL = 1024 + Q_BYTES + SLOTS * SLOT_BYTES + P_BYTES + 256;
  static constexpr int O_COL = 0, S_COL = 320;        // TMEM columns
};

// MC: CTA pairs (cluster of 2 along the query-tile axis, same frame) share every
// K/V^T ring slot: each CTA TMA-loads half of the slot and multicasts it to both,
// and a slot is refilled only after both CTAs' MMAs released it -- half the L2
// traffic per query tile.
template <int D, bool MC>
__global__ void __launch_bounds__(THREADS, 1)
    flash_kernel(const __grid_constant__ Params p, const __grid_constant__ CUtensorMap mQ,
                 const __grid_constant__ CUtensorMap mK, const __grid_constant__ CUtensorMap mV) {
  using L = Layout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;
  uint8_t* sRing = sQ + L::Q_BYTES;
  uint8_t* sP = sRing + SLOTS * L::SLOT_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + L::P_BYTES);
  uint64_t* q_full = bars;              // 1
  uint64_t* r_full = bars + 1;          // SLOTS
  uint64_t* r_empty = r_full + SLOTS;   // SLOTS
  uint64_t* s_full = r_empty + SLOTS;   // 2
  uint64_t* s_empty = s_full + 2;       // 2
  uint64_t* p_full = s_empty + 2;       // 1
  uint64_t* o_done = p_full + 1;        // 1
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, f = blockIdx.y;
  const int q0 = qt * BQ;
  const int nkv = p.n_kv;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < SLOTS; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], MC ? 2 : 1);   // both CTAs of the pair must release a shared slot
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 4);
    }
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
  if (MC) cluster_sync();   // peer barriers initialised before any multicast / remote arrive
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t crank = MC ? cluster_rank() : 0;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(q_full, L::Q_BYTES);
      for (int c = 0; c < L::NCH; ++c) tma3(&mQ, q_full, sQ + c * BQ * 128, c * 64, q0, f);
      // ring order: K_0, then (K_{j+1}, V_j) for j = 0..nkv-1 (K_nkv skipped)
      int slot = 0;
      uint32_t ph = 0;
      const int n_items = 2 * nkv;
      for (int item = 0; item < n_items; ++item) {
        int j;
        bool k_item;
        if (item == 0) {
          k_item = true;
          j = 0;
        } else if (item % 2 == 1) {
          // item 2t-1 -> K_t (t < nkv) else V_{t-1}
          const int t = (item + 1) / 2;
          if (t < nkv) {
            k_item = true;
            j = t;
          } else {
            k_item = false;
            j = t - 1;
          }
        } else {
          // item 2t -> V_{t-1}
          k_item = false;
          j = item / 2 - 1;
        }
        mbar_wait(&r_empty[slot], ph ^ 1);
        mbar_expect_tx(&r_full[slot], L::SLOT_BYTES);
        uint8_t* dst = sRing + slot * L::SLOT_BYTES;
        if (MC) {
          // my half of the slot, multicast to both CTAs (the peer loads the other half)
          if (k_item) {
            const int c0 = crank == 0 ? 0 : (L::NCH + 1) / 2, c1 = crank == 0 ? (L::NCH + 1) / 2 : L::NCH;
            for (int c = c0; c < c1; ++c)
              tma3_mc(&mK, &r_full[slot], dst + c * BKV * 128, c * 64, j * BKV, f, 0x3);
          } else {
            tma3_mc(&mV, &r_full[slot], dst + crank * (D / 2) * 128, j * BKV, crank * (D / 2), f, 0x3);
          }
        } else if (k_item) {
          for (int c = 0; c < L::NCH; ++c) tma3(&mK, &r_full[slot], dst + c * BKV * 128, c * 64, j * BKV, f);
        } else {
          tma3(&mV, &r_full[slot], dst, j * BKV, 0, f);
          tma3(&mV, &r_full[slot], dst + (D / 2) * 128, j * BKV, D / 2, f);
        }
        if (++slot == SLOTS) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc(BKV), idO = idesc(D / 2);
      mbar_wait(q_full, 0);
      fence_after();
      const uint64_t qd = sdesc(smem_u32(sQ));
      const uint64_t pd = sdesc(smem_u32(sP));
      int slot = 0;
      uint32_t ph = 0;
      auto issue_S = [&](int j) {
        const int sb = j & 1;
        mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        mbar_wait(&r_full[slot], ph);
        fence_after();
        // descriptors built once; every MMA only adds a constant to the address field
        const uint64_t kd = sdesc(smem_u32(sRing + slot * L::SLOT_BYTES));
        const uint32_t d = tmem + L::S_COL + sb * BKV;
#pragma unroll
        for (int c = 0; c < L::NCH; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma(d, qd + (uint64_t)((c * BQ * 128 + k * 32) >> 4), kd + (uint64_t)((c * BKV * 128 + k * 32) >> 4), idS,
                (c | k) != 0);
        if (MC) commit_mc(&r_empty[slot], 0x3);
        else commit(&r_empty[slot]);
        commit(&s_full[sb]);
        if (++slot == SLOTS) {
          slot = 0;
          ph ^= 1;
        }
      };
      auto issue_PV = [&](int j) {
        mbar_wait(p_full, j & 1);
        mbar_wait(&r_full[slot], ph);
        fence_after();
        const uint64_t vd = sdesc(smem_u32(sRing + slot * L::SLOT_BYTES));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mma(tmem + L::O_COL, pd + (uint64_t)(k * 2), vd + (uint64_t)(k * 2), idO, (j | k) != 0);
          mma(tmem + L::O_COL + D / 2, pd + (uint64_t)(k * 2), vd + (uint64_t)(((D / 2) * 128 + k * 32) >> 4), idO,
              (j | k) != 0);
        }
        if (MC) commit_mc(&r_empty[slot], 0x3);
        else commit(&r_empty[slot]);
        commit(o_done);
        if (++slot == SLOTS) {
          slot = 0;
          ph ^= 1;
        }
      };
      issue_S(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_S(j + 1);
        issue_PV(j);
      }
    }
  } else {
    // ================= softmax + epilogue (128 threads, one query row each) =================
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    const float c = p.scale_log2;
    // P tile row address pieces (SW128 K-major: 16B chunk index XOR row%8)
    uint8_t* prow = sP + (row >> 3) * 1024 + (row & 7) * 128;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      fence_after();
      uint32_t r[64];
      tld32(tmem + lane_off + L::S_COL + sb * BKV, r);
      tld32(tmem + lane_off + L::S_COL + sb * BKV + 32, r + 32);
      tld_wait();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      float s[64];
      float mb = -INFINITY;
      const int kbase = j * BKV;
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        s[e] = (kbase + e < p.HW) ? __uint_as_float(r[e]) * c : -INFINITY;
        mb = fmaxf(mb, s[e]);
      }
      // lazy rescale: only when the max grows by more than 8 (x256)
      bool need = false;
      float corr = 1.f;
      if (j == 0) {
        m_run = mb;
      } else if (mb > m_run + 8.f) {
        need = true;
        corr = exp2f(m_run - mb);
        m_run = mb;
      }
      // PV_{j-1} must be done before P is overwritten and before O is touched
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);
        fence_after();
      }
      if (__any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int cc = 0; cc < D; cc += 32) {
          uint32_t o[32];
          tld32(tmem + lane_off + L::O_COL + cc, o);
          tld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tst32(tmem + lane_off + L::O_COL + cc, o);
        }
        tst_wait();
      }
      l_run *= corr;
      float ls = 0.f;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        float pv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          pv[e] = exp2f(s[ch * 8 + e] - m_run);
          ls += pv[e];
        }
        bf16x8 packed = pack8(pv);
        *reinterpret_cast<bf16x8*>(prow + ((ch ^ (row & 7)) << 4)) = packed;
      }
      l_run += ls;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 rows
    mbar_wait(o_done, (nkv - 1) & 1);
    fence_after();
    const float inv = 1.f / l_run;
    const int qrow = q0 + row;
    const bool valid = qrow < p.HW;
    bf16* dst = reinterpret_cast<bf16*>(p.out.ptr) + ((int64_t)f * p.out.ostride + qrow) * p.out.ld;
#pragma unroll 1
    for (int cc = 0; cc < D; cc += 32) {
      uint32_t o[32];
      tld32(tmem + lane_off + L::O_COL + cc, o);
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
  if (MC) cluster_sync();   // no CTA leaves while its peer may still multicast into it
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
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(flash_kernel<D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(flash_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  const int qt = (p.HW + BQ - 1) / BQ;
  if (qt >= 2) {
    // CTA pairs share K/V: grid.x rounded up to even (a padding tile only masks its rows)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)((qt + 1) / 2 * 2), (unsigned)p.frames, 1);
    cfg.blockDim = dim3(THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, flash_kernel<D, true>, p, q, k, v);
  } else {
    dim3 grid(qt, p.frames);
    flash_kernel<D, false><<<grid, THREADS, smem, st>>>(p, q, k, v);
  }
  return launch_status("sf_spatial_attention_core");
}

}  // namespace fa
}  // namespace sf

namespace sf {
sf_status flash2_launch(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int frames, int HW, int C,
                        float scale, cudaStream_t st);
sf_status flash3_launch(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int frames, int HW, int C,
                        float scale, cudaStream_t st);
bool flash3_supported(int C);
}
using namespace sf;

extern "C" int32_t sf_flash_supported(int32_t HW, int32_t C) {
  return (C == 320 || C == 256 || C == 192 || C == 128) && HW >= 64 && fa::encode_fn() != nullptr;
}

extern "C" sf_status sf_spatial_attention_core(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int32_t frames,
                                               int32_t HW, int32_t C, float scale, void* stream) {
  SF_CHECK_ARG(frames >= 1 && HW >= 1, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(sf_flash_supported(HW, C), SF_ERR_UNSUPPORTED, "fused attention needs C in {128,192,256,320}");
  SF_CHECK_ARG(view_vec8_ok(q) && view_vec8_ok(k) && view_vec8_ok(out) && aligned16(vt) && HW % 8 == 0,
               SF_ERR_PARAM, "operands must be 16-byte aligned, HW % 8 == 0");
  SF_CHECK_ARG(q.ld == k.ld, SF_ERR_PARAM, "q and k must share a row stride");
  fa::Params p{};
  p.HW = HW;
  p.frames = frames;
  p.n_kv = (HW + fa::BKV - 1) / fa::BKV;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.out = out;
  const uint64_t es = 2;
  const uint64_t qst = (uint64_t)(q.ostride ? q.ostride : HW) * q.ld * es;
  CUtensorMap mq, mk, mv;
  SF_CHECK_ARG(fa::enc3(&mq, q.ptr, C, HW, frames, q.ld * es, qst, 64, fa::BQ), SF_ERR_CUDA, "tensor map Q");
  SF_CHECK_ARG(fa::enc3(&mk, k.ptr, C, HW, frames, k.ld * es, qst, 64, fa::BKV), SF_ERR_CUDA, "tensor map K");
  SF_CHECK_ARG(fa::enc3(&mv, vt, HW, C, frames, (uint64_t)HW * es, (uint64_t)C * HW * es, 64, C / 2), SF_ERR_CUDA,
               "tensor map V");
  cudaStream_t st = (cudaStream_t)stream;
  static const char* ver = getenv("SF_FLASH");   // "1" / "2" force an older kernel (A/B runs)
  const int v = ver ? atoi(ver) : 3;
  if (v >= 3 && flash3_supported(C) && (HW + 127) / 128 >= 2) return flash3_launch(q, k, vt, out, frames, HW, C, scale, st);
  if (v >= 2) return flash2_launch(q, k, vt, out, frames, HW, C, scale, st);
  switch (C) {
    case 320: return fa::launch<320>(p, mq, mk, mv, st);
    case 256: return fa::launch<256>(p, mq, mk, mv, st);
    case 192: return fa::launch<192>(p, mq, mk, mv, st);
    default: return fa::launch<128>(p, mq, mk, mv, st);
  }
}
