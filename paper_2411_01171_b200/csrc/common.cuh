// Shared helpers for the sm_100a kernels of sliceflow_b200.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/sliceflow_b200.h"

namespace sf {

typedef __nv_bfloat16 bf16;
typedef __nv_bfloat162 bf162;

// thread-local last error text (sf_last_error)
void set_error(const std::string& msg);

#define SF_CHECK_ARG(cond, code, msg)                   \
  do {                                                  \
    if (!(cond)) {                                      \
      ::sf::set_error(std::string(__func__) + ": " + (msg)); \
      return (code);                                    \
    }                                                   \
  } while (0)

inline sf_status launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return SF_ERR_CUDA;
  }
  return SF_OK;
}

// Row (o, i) of a two-level view.
template <typename T>
__device__ __forceinline__ T* row_ptr(const sf_view_t& v, int64_t o, int64_t i) {
  return reinterpret_cast<T*>(v.ptr) + (o * v.ostride + i) * v.ld;
}

__device__ __forceinline__ float silu_f(float x) {
  // x * sigmoid(x) = 0.5x + 0.5x * tanh(0.5x) (kernels.py:247-253): one MUFU op (tanh.approx,
  // abs error ~2^-11, far below the bf16 rounding of every SiLU output here) instead of an
  // ex2 + a reciprocal -- SiLU made the fused GroupNorm apply MUFU-bound (69 vs 60 us at L0)
  float t;
  const float h = 0.5f * x;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
  return fmaf(h, t, h);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}

// 8 x bf16 <-> 8 x float through one 16-byte access.  Backed by a uint4 so a
// copy is one LDG/STG.128 (bf162 members have user-defined copy operators,
// which made struct copies member-wise 4-byte accesses).
struct alignas(16) bf16x8 {
  uint4 u;
};
__device__ __forceinline__ bf162 bf2_of(uint32_t w) { return *reinterpret_cast<const bf162*>(&w); }
__device__ __forceinline__ uint32_t u32_of(bf162 h) { return *reinterpret_cast<const uint32_t*>(&h); }
__device__ __forceinline__ void unpack8(const bf16x8& v, float* f) {
  const uint32_t w[4] = {v.u.x, v.u.y, v.u.z, v.u.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 t = __bfloat1622float2(bf2_of(w[j]));
    f[2 * j] = t.x;
    f[2 * j + 1] = t.y;
  }
}
__device__ __forceinline__ bf16x8 pack8(const float* f) {
  bf16x8 v;
  v.u.x = u32_of(__floats2bfloat162_rn(f[0], f[1]));
  v.u.y = u32_of(__floats2bfloat162_rn(f[2], f[3]));
  v.u.z = u32_of(__floats2bfloat162_rn(f[4], f[5]));
  v.u.w = u32_of(__floats2bfloat162_rn(f[6], f[7]));
  return v;
}

// Programmatic dependent launch (PDL).  Every kernel of this library starts with
// griddep_wait() -- block until the grid this one depends on has completed and its
// writes are visible (a no-op when launched without PDL) -- before touching global
// memory, then griddep_trigger() so the next kernel in the stream can be scheduled
// while this one runs (its blocks park in their own griddep_wait).  All launches go
// through launch_k, which sets the stream-serialisation attribute when SF_PDL=1.
// Off by default: measured on B200 inside the CUDA-graph run it cost ~1 % (79.2 vs
// 80.2 steps/s) -- the parked blocks hold SM slots and the launch gaps it hides are small.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SF_PDL");
    on = e && e[0] == '1';
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
inline bool view_vec8_ok(const sf_view_t& v) { return aligned16(v.ptr) && (v.ld % 8) == 0; }

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (!n) n = 148;
  }
  return n;
}

// Row tiling of a CONV3X3 implicit GEMM over one frame (gemm_tc.cu): 128-row tiles of
// w_t x h_t pixels (w_t = the largest power of two <= min(W, 128)); when H % h_t = rem divides
// h_t, the last rem rows of h_t / rem consecutive frames form one *tail tile* per x-tile
// (SF_GEMM_TAIL=0 turns that off, and the last band then overhangs the frame).  The epilogue's
// GroupNorm partials use one split per 64-row half of a main tile and one per tail tile:
// splits per frame = 2 * tiles_x * tiles_y + (tail ? tiles_x : 0).
struct ConvTiling {
  int w_t, h_t, tiles_x, tiles_y, tail_rows, tail_fb;
  __host__ __device__ int gn_splits() const { return 2 * tiles_x * tiles_y + (tail_rows ? tiles_x : 0); }
};
inline ConvTiling conv_tiling(int H, int W) {
  ConvTiling t{};
  int p = 1;
  const int cap = W < 128 ? W : 128;
  while (p * 2 <= cap) p *= 2;
  t.w_t = p;
  t.h_t = 128 / p;
  t.tiles_x = (W + t.w_t - 1) / t.w_t;
  t.tiles_y = (H + t.h_t - 1) / t.h_t;
  const int rem = H % t.h_t;
  static const char* tail_env = getenv("SF_GEMM_TAIL");
  if (rem && t.h_t % rem == 0 && !(tail_env && tail_env[0] == '0')) {
    t.tail_rows = rem;
    t.tail_fb = t.h_t / rem;
    t.tiles_y = H / t.h_t;
  }
  return t;
}

}  // namespace sf
