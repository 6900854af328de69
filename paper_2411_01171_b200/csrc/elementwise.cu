// HBM-bound kernels of the sliceflow path: norms, SiLU, add, resampling,
// copies, softmax rows, latent-edge convolutions, similarity dot products.
//
// All bf16 activation kernels move 16-byte vectors (8 channels) and require
// C % 8 == 0 and 16-byte aligned rows; reductions are fixed-order (no float
// atomics) so results are bit-reproducible run to run.
#include "common.cuh"

#include <algorithm>
#include <cstdlib>

#include <cmath>
#include <mutex>

namespace sf {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

// ---------------------------------------------------------------------------
// GroupNorm (kernels.py:228-237)
// ---------------------------------------------------------------------------

static int gn_splits(int frames, int n_inner) {
  // ~2 CTAs per SM: each partial is a full (C) row of fp64 sums the finalize
  // pass has to walk, so long CTAs beat many light ones (measured on B200)
  static const int per_sm = getenv("SF_GN_CTAS") ? atoi(getenv("SF_GN_CTAS")) : 2;        // tuning knobs
  static const int min_rows = getenv("SF_GN_MINROWS") ? atoi(getenv("SF_GN_MINROWS")) : 64;
  // rounded down: frames x splits <= per_sm x SMs, so no SM runs a lone extra block at the end
  // (tools/gn_bench.py: C3 L0 50.2 -> 48.2 us, the L0 concat 105 -> 101 us)
  int want = (per_sm * num_sms()) / frames;
  int most = (n_inner + min_rows - 1) / min_rows;        // >= min_rows rows per CTA
  int s = want < most ? want : most;
  return s < 1 ? 1 : s;
}

// partial[frame][split][c] = (sum x, sum x^2) over the split's rows, fp64
#ifndef GN_UNROLL
#define GN_UNROLL 8   // 16-byte loads in flight per thread (tuning: -DGN_UNROLL=n)
#endif
constexpr int GN_U = GN_UNROLL;
__global__ void __launch_bounds__(256, 4) gn_partial_kernel(sf_view_t x, int n_inner, int C, int splits,
                                                            double2* partial) {
  griddep_wait();
  const int frame = blockIdx.x / splits, split = blockIdx.x % splits;
  const int nvec = C / 8;
  const int rows_per_iter = blockDim.x / nvec > 0 ? blockDim.x / nvec : 1;
  const int chunk = (n_inner + splits - 1) / splits;
  const int r0 = split * chunk, r1 = min(n_inner, r0 + chunk);
  extern __shared__ double2 red[];  // [rows_per_iter][C] when nvec <= blockDim
  const int lane_v = nvec <= (int)blockDim.x ? (int)threadIdx.x % nvec : (int)threadIdx.x;
  const int lane_r = nvec <= (int)blockDim.x ? (int)threadIdx.x / nvec : 0;
  const bool active = nvec <= (int)blockDim.x ? lane_r < rows_per_iter : true;
  for (int vbase = lane_v; vbase < nvec; vbase += (nvec <= (int)blockDim.x ? nvec : blockDim.x)) {
    float s[8], q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = q[j] = 0.f;
    if (active) {
      // GN_U independent 16-byte loads in flight per thread, then fp32 partials -> fp64
      int r = r0 + lane_r;
      for (; r + (GN_U - 1) * rows_per_iter < r1; r += GN_U * rows_per_iter) {
        bf16x8 v[GN_U];
#pragma unroll
        for (int u = 0; u < GN_U; ++u)
          v[u] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, frame, r + u * rows_per_iter) + vbase * 8);
        float fs[8], fq[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) fs[j] = fq[j] = 0.f;
#pragma unroll
        for (int u = 0; u < GN_U; ++u) {
          float f[8];
          unpack8(v[u], f);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            fs[j] += f[j];
            fq[j] += f[j] * f[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[j] += fs[j];
          q[j] += fq[j];
        }
      }
      for (; r < r1; r += rows_per_iter) {
        bf16x8 v = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, frame, r) + vbase * 8);
        float f[8];
        unpack8(v, f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[j] += f[j];
          q[j] += f[j] * f[j];
        }
      }
    }
    if (nvec <= (int)blockDim.x) {
      if (active) {
#pragma unroll
        for (int j = 0; j < 8; ++j) red[lane_r * C + vbase * 8 + j] = make_double2((double)s[j], (double)q[j]);
      }
      __syncthreads();
      if (lane_r == 0) {
        for (int j = 0; j < 8; ++j) {
          double ss = 0, qq = 0;
          for (int rr = 0; rr < rows_per_iter; ++rr) {
            double2 t = red[rr * C + vbase * 8 + j];
            ss += t.x;
            qq += t.y;
          }
          partial[((int64_t)frame * splits + split) * C + vbase * 8 + j] = make_double2(ss, qq);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        partial[((int64_t)frame * splits + split) * C + vbase * 8 + j] = make_double2((double)s[j], (double)q[j]);
    }
  }
}

// mean / rstd from per-split (sum, sum sq) partials [frame][split][C] (fp64 from gn_partial_kernel,
// fp32 from a conv epilogue / sf_conv_gn_partials).  Block = (frame, a run of gpb whole groups =
// CH channels) with SPL split lanes per channel: thread (l, c) sums splits l, l + SPL, ... of
// channel c in fp64 (independent loads in flight), the SPL lane sums are added in lane order, then
// one warp per group adds its channels.  Fixed summation order: bitwise reproducible.  (One thread
// per channel walking all splits was latency-bound: 144 splits x 320 channels at C3 L0 took 23 us
// in 50 blocks.)
template <typename T>
__global__ void __launch_bounds__(256) gn_finalize_kernel(const T* __restrict__ partial, int splits, int C,
                                                          int groups, int gpb, int spl, int64_t count, float eps,
                                                          float* mean, float* rstd) {
  griddep_wait();
  extern __shared__ double2 tot[];   // [spl][CH]
  const int cg = C / groups, CH = gpb * cg;
  const int frame = blockIdx.y, g0 = blockIdx.x * gpb;
  const int ng = min(gpb, groups - g0), nch = ng * cg;
  const T* base = partial + (int64_t)frame * splits * C + (int64_t)g0 * cg;
  for (int t = threadIdx.x; t < spl * CH; t += blockDim.x) {
    const int l = t / CH, c = t % CH;
    double s = 0, q = 0;
    if (c < nch) {
      int sp = l;
      for (; sp + 3 * spl < splits; sp += 4 * spl) {
        T v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = base[(int64_t)(sp + u * spl) * C + c];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s += (double)v[u].x;
          q += (double)v[u].y;
        }
      }
      for (; sp < splits; sp += spl) {
        const T v = base[(int64_t)sp * C + c];
        s += (double)v.x;
        q += (double)v.y;
      }
    }
    tot[l * CH + c] = make_double2(s, q);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nch; c += blockDim.x) {
    double2 a = tot[c];
    for (int l = 1; l < spl; ++l) {
      a.x += tot[l * CH + c].x;
      a.y += tot[l * CH + c].y;
    }
    tot[c] = a;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int gi = warp; gi < ng; gi += blockDim.x >> 5) {
    double s = 0, q = 0;
    for (int c = lane; c < cg; c += 32) {
      s += tot[gi * cg + c].x;
      q += tot[gi * cg + c].y;
    }
    s = warp_sum_d(s);
    q = warp_sum_d(q);
    if (lane == 0) {
      const double mu = s / (double)count;
      double var = q / (double)count - mu * mu;
      if (var < 0) var = 0;
      const int o = frame * groups + g0 + gi;
      mean[o] = (float)mu;
      rstd[o] = (float)(1.0 / sqrt(var + (double)eps));
    }
  }
}

template <typename T>
static void launch_gn_finalize(const T* partial, int frames, int splits, int C, int groups, int64_t count, float eps,
                               float* mean, float* rstd, cudaStream_t st) {
  const int cg = C / groups;
  // split lanes: up to 16, as long as one block (256 threads) still holds a whole group
  int spl = 1;
  while (spl < 16 && spl * 2 <= splits && 256 / (spl * 2) >= cg) spl *= 2;
  const int CH = cg >= 256 / spl ? cg : (256 / spl) / cg * cg;
  const int gpb = CH / cg;
  const size_t smem = (size_t)spl * CH * sizeof(double2);
  if (smem > 48 * 1024) {
    static size_t set = 0;
    if (smem > set) {
      cudaFuncSetAttribute(gn_finalize_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      set = smem;
    }
  }
  launch_k(gn_finalize_kernel<T>, dim3((groups + gpb - 1) / gpb, frames), dim3(256), smem, st, partial, splits, C,
           groups, gpb, spl, count, eps, mean, rstd);
}

// GroupNorm partials of a CONV3X3 output as a separate pass, in the layout and summation order
// of the tcgen05 GEMM epilogue's (gemm_tc.cu gn_tile_partials): the mma.sync backend's
// counterpart, and the checker of the fused partials (identical bits).  Block = (split, frame),
// thread = a column pair.
__global__ void __launch_bounds__(128) conv_gn_partials_kernel(sf_view_t y, int H, int W, int N, ConvTiling ct,
                                                               float2* part) {
  griddep_wait();
  const int s = blockIdx.x, fr = blockIdx.y, splits = ct.gn_splits();
  const int n_main = 2 * ct.tiles_x * ct.tiles_y;
  int x0, y0, r0, nrows;
  if (s < n_main) {
    const int tile = s >> 1;
    x0 = (tile % ct.tiles_x) * ct.w_t;
    y0 = (tile / ct.tiles_x) * ct.h_t;
    r0 = (s & 1) * 64;
    nrows = 64;
  } else {
    x0 = (s - n_main) * ct.w_t;
    y0 = ct.tiles_y * ct.h_t;
    r0 = 0;
    nrows = ct.tail_rows * ct.w_t;
  }
  for (int c2 = threadIdx.x; 2 * c2 < N; c2 += blockDim.x) {
    // row r -> accumulator r % 4, combined (0+1)+(2+3): gemm_tc.cu gn_tile_partials' order
    float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
    float q0[4] = {0.f, 0.f, 0.f, 0.f}, q1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < nrows; ++r) {
      const int yy = y0 + (r0 + r) / ct.w_t, xx = x0 + (r0 + r) % ct.w_t;
      if (yy < H && xx < W) {
        const float2 f =
            __bfloat1622float2(*reinterpret_cast<const bf162*>(row_ptr<const bf16>(y, fr, (int64_t)yy * W + xx) + 2 * c2));
        const int u = r & 3;
        a0[u] += f.x;
        q0[u] = fmaf(f.x, f.x, q0[u]);
        a1[u] += f.y;
        q1[u] = fmaf(f.y, f.y, q1[u]);
      }
    }
    part[((int64_t)fr * splits + s) * N + 2 * c2] =
        make_float2((a0[0] + a0[1]) + (a0[2] + a0[3]), (q0[0] + q0[1]) + (q0[2] + q0[3]));
    part[((int64_t)fr * splits + s) * N + 2 * c2 + 1] =
        make_float2((a1[0] + a1[1]) + (a1[2] + a1[3]), (q1[0] + q1[1]) + (q1[2] + q1[3]));
  }
}

sf_status conv_gn_partials(sf_view_t y, int frames, int H, int W, int N, void* part, cudaStream_t st) {
  const ConvTiling ct = conv_tiling(H, W);
  launch_k(conv_gn_partials_kernel, dim3((unsigned)ct.gn_splits(), (unsigned)frames), dim3(128), 0, st, y, H, W, N,
           ct, (float2*)part);
  return launch_status("conv_gn_partials");
}

// Small planes (deep levels, n_inner <= GN_DIRECT_MAX_ROWS): ONE launch, one block per (frame,
// run of gpb whole groups = W channels): 8-channel vectors x rows_per_iter row lanes read the
// block's rows (GN_U loads in flight), fp32 per thread -> fp64 per channel in shared memory ->
// fp64 per group -> mean / rstd.  Fixed order: bitwise reproducible.  (The split + finalize pair
// costs two dependent launches over 9-37 MB here: 17-27 us at 0.5-1.4 TB/s.)
constexpr int GN_DIRECT_MAX_ROWS = 1024;
__global__ void __launch_bounds__(256) gn_stats_direct_kernel(sf_view_t x, int n_inner, int C, int groups, int gpb,
                                                              float eps, float* mean, float* rstd) {
  griddep_wait();
  extern __shared__ double2 red[];   // [rows_per_iter][W], then [W] channel totals in row 0
  const int cg = C / groups, W = gpb * cg, nv = W / 8;
  const int frame = blockIdx.y, g0 = blockIdx.x * gpb, c0 = g0 * cg;
  const int rpi = (int)blockDim.x / nv;
  const int v = threadIdx.x % nv, lr = threadIdx.x / nv;
  if (lr < rpi) {
    float s[8], q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = q[j] = 0.f;
    const bf16* base = row_ptr<const bf16>(x, frame, 0) + c0 + v * 8;
    int r = lr;
    for (; r + (GN_U - 1) * rpi < n_inner; r += GN_U * rpi) {
      bf16x8 in[GN_U];
#pragma unroll
      for (int u = 0; u < GN_U; ++u) in[u] = *reinterpret_cast<const bf16x8*>(base + (int64_t)(r + u * rpi) * x.ld);
#pragma unroll
      for (int u = 0; u < GN_U; ++u) {
        float f[8];
        unpack8(in[u], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[j] += f[j];
          q[j] += f[j] * f[j];
        }
      }
    }
    for (; r < n_inner; r += rpi) {
      float f[8];
      unpack8(*reinterpret_cast<const bf16x8*>(base + (int64_t)r * x.ld), f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[j] += f[j];
        q[j] += f[j] * f[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) red[lr * W + v * 8 + j] = make_double2((double)s[j], (double)q[j]);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < W; c += blockDim.x) {
    double ss = 0, qq = 0;
    for (int rr = 0; rr < rpi; ++rr) {
      const double2 t = red[rr * W + c];
      ss += t.x;
      qq += t.y;
    }
    red[c] = make_double2(ss, qq);   // row 0 is only read by this thread above
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ng = min(gpb, groups - g0);
  const double count = (double)n_inner * cg;
  for (int gi = warp; gi < ng; gi += blockDim.x >> 5) {
    double ss = 0, qq = 0;
    for (int c = lane; c < cg; c += 32) {
      ss += red[gi * cg + c].x;
      qq += red[gi * cg + c].y;
    }
    ss = warp_sum_d(ss);
    qq = warp_sum_d(qq);
    if (lane == 0) {
      const double mu = ss / count;
      double var = qq / count - mu * mu;
      if (var < 0) var = 0;
      const int o = frame * groups + g0 + gi;
      mean[o] = (float)mu;
      rstd[o] = (float)(1.0 / sqrt(var + (double)eps));
    }
  }
}

// groups per block of the direct statistics kernel: about 160 channels (20 vectors x 12 row lanes)
// and a multiple of 8 channels; 0 = not applicable
static int gn_direct_gpb(int C, int groups, int n_inner) {
  if (n_inner > GN_DIRECT_MAX_ROWS) return 0;
  const int cg = C / groups;
  for (int gpb = std::max(1, 160 / cg); gpb >= 1; --gpb)
    if ((gpb * cg) % 8 == 0 && gpb * cg <= 256 * 8 && groups % gpb == 0) return gpb;
  return 0;
}

// y = act((x - mean[f][g]) * (rstd[f][g] * gamma[c]) + beta[c]).  Persistent: each
// block takes an equal contiguous share of all frames*n_inner rows (no tail wave);
// each thread owns one 8-channel vector (mean / scale / shift in registers, reloaded
// when its rows cross into the next frame) and walks rows with 8 loads in flight.
__global__ void __launch_bounds__(256) gn_apply_kernel(sf_view_t x, sf_view_t y, int frames, int n_inner, int C,
                                                       int groups, const float* __restrict__ mean,
                                                       const float* __restrict__ rstd,
                                                       const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, int act) {
  griddep_wait();
  const int cg = C / groups, nvec = C / 8;
  const int rpi = nvec <= (int)blockDim.x ? (int)blockDim.x / nvec : 1;   // rows per iteration
  const int64_t total = (int64_t)frames * n_inner;
  const int64_t r0 = total * blockIdx.x / gridDim.x, r1 = total * (blockIdx.x + 1) / gridDim.x;
  for (int v = nvec <= (int)blockDim.x ? (int)threadIdx.x % nvec : (int)threadIdx.x; v < nvec;
       v += nvec <= (int)blockDim.x ? nvec : (int)blockDim.x) {
    const int lr = nvec <= (int)blockDim.x ? (int)threadIdx.x / nvec : 0;
    if (lr >= rpi) return;
    // split this block's rows at frame boundaries: per segment one frame's tables
    for (int64_t seg = r0; seg < r1;) {
      const int f = (int)(seg / n_inner);
      const int64_t seg_end = min(r1, (int64_t)(f + 1) * n_inner);
      const int i0 = (int)(seg - (int64_t)f * n_inner), i1 = (int)(seg_end - (int64_t)f * n_inner);
      seg = seg_end;
      // y = x * ss + bb with ss = rstd * gamma, bb = beta - mean * ss (one FMA per element)
      float ss[8], bb[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = v * 8 + j, g = c / cg;
        ss[j] = __ldg(rstd + f * groups + g) * __ldg(gamma + c);
        bb[j] = fmaf(-__ldg(mean + f * groups + g), ss[j], __ldg(beta + c));
      }
      const bf16* src = row_ptr<const bf16>(x, f, 0) + v * 8;
      bf16* dst = row_ptr<bf16>(y, f, 0) + v * 8;
      const int64_t xld = x.ld, yld = y.ld;
      constexpr int U = 8;
      int i = i0 + lr;
      for (; i + (U - 1) * rpi < i1; i += U * rpi) {
        bf16x8 in[U];
#pragma unroll
        for (int u = 0; u < U; ++u) in[u] = *reinterpret_cast<const bf16x8*>(src + (int64_t)(i + u * rpi) * xld);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float fv[8];
          unpack8(in[u], fv);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float t = fmaf(fv[j], ss[j], bb[j]);
            fv[j] = act ? silu_f(t) : t;
          }
          *reinterpret_cast<bf16x8*>(dst + (int64_t)(i + u * rpi) * yld) = pack8(fv);
        }
      }
      for (; i < i1; i += rpi) {
        float fv[8];
        unpack8(*reinterpret_cast<const bf16x8*>(src + (int64_t)i * xld), fv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float t = fmaf(fv[j], ss[j], bb[j]);
          fv[j] = act ? silu_f(t) : t;
        }
        *reinterpret_cast<bf16x8*>(dst + (int64_t)i * yld) = pack8(fv);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// LayerNorm over channels (kernels.py:240-244): L lanes per row (32/L rows per
// warp), VPL 16-byte vectors per lane, two-pass (mean, then mean of squared
// deviations) from registers like the reference.
// ---------------------------------------------------------------------------
template <int L, int VPL>
__global__ void __launch_bounds__(256, VPL <= 5 ? 4 : 3) layer_norm_kernel(sf_view_t x, sf_view_t y, int n_outer,
                                                                         int n_inner, int C,
                                                                         const float* __restrict__ gamma,
                                                                         const float* __restrict__ beta, float eps,
                                                                         int act, float2* __restrict__ stats) {
  griddep_wait();
  // gamma / beta staged in shared memory once per block: the per-row parameter reads were 4
  // L1 loads per 16-byte data vector, competing with the data stream
  extern __shared__ float4 ln_par[];   // [2][C/4]
  for (int i = threadIdx.x; !stats && i < C / 4; i += blockDim.x) {
    ln_par[i] = __ldg(reinterpret_cast<const float4*>(gamma) + i);
    ln_par[C / 4 + i] = __ldg(reinterpret_cast<const float4*>(beta) + i);
  }
  __syncthreads();
  const float4* sg = ln_par;
  const float4* sb = ln_par + C / 4;
  constexpr int RPW = 32 / L;  // rows per warp
  const int64_t rows = (int64_t)n_outer * n_inner;
  const int lane = threadIdx.x & 31, sub = lane % L, grp = lane / L;
  const int nvec = C / 8;
  const int64_t warps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // the row's vectors stay packed (bf16) in registers and are unpacked per pass: half the
  // registers of fp32 copies, so more warps (and loads) are resident per SM
  auto load = [&](int64_t base, bf16x8* v) {
    const int64_t row = base + grp;
    if (row < rows) {
      const bf16* src = row_ptr<const bf16>(x, (int)(row / n_inner), (int)(row % n_inner));
#pragma unroll
      for (int k = 0; k < VPL; ++k)
        if (sub + L * k < nvec) v[k] = *reinterpret_cast<const bf16x8*>(src + (sub + L * k) * 8);
    }
  };
  int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * RPW;
  bf16x8 cur[VPL];
  if (base < rows) load(base, cur);
  for (; base < rows; base += warps_total * RPW) {
    const int64_t row = base + grp;
    const bool live = row < rows;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (live && sub + L * k < nvec) {
        float f[8];
        unpack8(cur[k], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += f[j];
      }
    }
#pragma unroll
    for (int m = L / 2; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    const float mu = s / C;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (live && sub + L * k < nvec) {
        float f[8];
        unpack8(cur[k], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = f[j] - mu;
          q += d * d;
        }
      }
    }
#pragma unroll
    for (int m = L / 2; m > 0; m >>= 1) q += __shfl_xor_sync(0xffffffffu, q, m);
    const float rs = rsqrtf(q / C + eps);
    if (stats) {
      // statistics only (LayerNorm folded into the next GEMM, sf_gemm_args.rowstats)
      if (live && sub == 0) stats[row] = make_float2(rs, -mu * rs);
    } else if (live) {
      bf16* dst = row_ptr<bf16>(y, (int)(row / n_inner), (int)(row % n_inner));
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        const int v = sub + L * k;
        if (v < nvec) {
          const float4 g0 = sg[2 * v], g1 = sg[2 * v + 1];
          const float4 b0 = sb[2 * v], b1 = sb[2 * v + 1];
          const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
          const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          float f[8], g[8];
          unpack8(cur[k], f);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float t = (f[j] - mu) * rs * gg[j] + bb[j];
            g[j] = act ? silu_f(t) : t;
          }
          *reinterpret_cast<bf16x8*>(dst + v * 8) = pack8(g);
        }
      }
    }
    if (base + warps_total * RPW < rows) load(base + warps_total * RPW, cur);
  }
}

// ---------------------------------------------------------------------------
// elementwise on row views
// ---------------------------------------------------------------------------
enum { EW_SILU = 0, EW_ADD = 1, EW_COPY = 2 };

template <int OP>
__global__ void rows_ew_kernel(sf_view_t a, sf_view_t b, sf_view_t y, int n_outer, int n_inner, int C,
                               int b_bcast) {
  griddep_wait();
  const int nvec = C / 8;
  const int64_t total = (int64_t)n_outer * n_inner * nvec;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int v = idx % nvec;
    int64_t row = idx / nvec;
    int o = row / n_inner, i = row % n_inner;
    bf16x8 va = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(a, o, i) + v * 8);
    if (OP == EW_COPY) {
      *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, o, i) + v * 8) = va;
      continue;
    }
    float f[8];
    unpack8(va, f);
    if (OP == EW_SILU) {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = silu_f(f[j]);
    } else {
      float g[8];
      unpack8(*reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(b, o, b_bcast ? 0 : i) + v * 8), g);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += g[j];
    }
    *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, o, i) + v * 8) = pack8(f);
  }
}

__global__ void copy_rows_scalar_kernel(sf_view_t x, sf_view_t y, int n_outer, int n_inner, int C) {
  griddep_wait();
  const int64_t total = (int64_t)n_outer * n_inner * C;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int c = idx % C;
    int64_t row = idx / C;
    int o = row / n_inner, i = row % n_inner;
    row_ptr<bf16>(y, o, i)[c] = row_ptr<const bf16>(x, o, i)[c];
  }
}

__global__ void downsample_kernel(sf_view_t x, sf_view_t y, int frames, int H, int W, int C) {
  griddep_wait();
  const int nvec = C / 8, Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)frames * Ho * Wo * nvec;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int v = idx % nvec;
    int64_t p = idx / nvec;
    int xo = p % Wo, yo = (p / Wo) % Ho, f = p / ((int64_t)Wo * Ho);
    float a[8], b[8], c[8], d[8], r[8];
    unpack8(*reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, (2 * yo) * W + 2 * xo) + v * 8), a);
    unpack8(*reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, (2 * yo) * W + 2 * xo + 1) + v * 8), b);
    unpack8(*reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, (2 * yo + 1) * W + 2 * xo) + v * 8), c);
    unpack8(*reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, (2 * yo + 1) * W + 2 * xo + 1) + v * 8), d);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = (((a[j] + b[j]) + c[j]) + d[j]) * 0.25f;
    *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, yo * Wo + xo) + v * 8) = pack8(r);
  }
}

// nearest 2x upsample: one thread per input 16-byte vector, stored to its 2x2 output block
// (one load, four coalesced stores; 32-bit index math)
__global__ void upsample_kernel(sf_view_t x, sf_view_t y, int frames, int H, int W, int C) {
  griddep_wait();
  const int nvec = C / 8, Wo = 2 * W;
  const uint32_t total = (uint32_t)frames * H * W * nvec;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const uint32_t v = idx % nvec, p = idx / nvec;
    const uint32_t xi = p % W, t = p / W, yi = t % H, f = t / H;
    const bf16x8 val = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, (int64_t)yi * W + xi) + v * 8);
    const int64_t o = (int64_t)(2 * yi) * Wo + 2 * xi;
    *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o) + v * 8) = val;
    *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o + 1) + v * 8) = val;
    *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o + Wo) + v * 8) = val;
    *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o + Wo + 1) + v * 8) = val;
  }
}

// Resampling with GroupNorm partials (the statistics the next GroupNorm would otherwise take in a
// pass of its own; unet.py:221-244: down_blocks.i.downsample -> down_blocks.i+1.res.norm1, and the
// skip / upsampled halves of up_blocks.i.concat -> up_blocks.i.res.norm1).  Block = (split, frame):
// the split's contiguous range of COARSE pixels (the downsample's outputs, the upsample's inputs),
// thread = (row lane, 8-channel vector); fp32 sums per thread, row lanes combined in lane order in
// shared memory.  Partials land at part[(frame * splits + split) * ld + c0 + c] as float2 (sum,
// sum sq):
//   UP = 0: out_part = the stored (bf16-rounded) pooled output, in_part = the 4 input pixels read;
//   UP = 1: out_part = the 2x2 copies written (4 x the input's sums, exact in fp32).
template <int UP>
__global__ void __launch_bounds__(256) resample_gn_kernel(sf_view_t x, sf_view_t y, int H, int W, int C, int splits,
                                                          float2* out_part, int out_ld, int out_c0, float2* in_part,
                                                          int in_ld) {
  griddep_wait();
  extern __shared__ float4 rsm[];   // [rows_per_iter][C] (out sum, out sq, in sum, in sq)
  const int f = blockIdx.y, sp = blockIdx.x;
  const int nvec = C / 8;
  const int Wc = UP ? W : W / 2, coarse = UP ? H * W : (H / 2) * (W / 2);
  const int chunk = (coarse + splits - 1) / splits;
  const int p0 = sp * chunk, p1 = min(coarse, p0 + chunk);
  const bool fits = nvec <= (int)blockDim.x;
  const int rpi = fits ? blockDim.x / nvec : 1;
  const int lane_v = fits ? threadIdx.x % nvec : threadIdx.x, lane_r = fits ? threadIdx.x / nvec : 0;
  const bool active = lane_r < rpi;
  for (int vb = lane_v; vb < nvec; vb += fits ? nvec : blockDim.x) {
    float os[8], oq[8], is[8], iq[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) os[j] = oq[j] = is[j] = iq[j] = 0.f;
    if (active) {
      // U coarse pixels per iteration, all loads issued before the math (memory-level parallelism:
      // a block walks only its split's pixels)
      constexpr int U = UP ? 4 : 2;
      for (int pc0 = p0 + lane_r; pc0 < p1; pc0 += U * rpi) {
        if (UP) {
          bf16x8 val[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int pc = pc0 + u * rpi;
            if (pc < p1)
              val[u] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, (int64_t)(pc / Wc) * W + pc % Wc) +
                                                        vb * 8);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int pc = pc0 + u * rpi;
            if (pc >= p1) break;
            const int xc = pc % Wc, yc = pc / Wc;
            const int64_t o = (int64_t)(2 * yc) * (2 * W) + 2 * xc;
            *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o) + vb * 8) = val[u];
            *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o + 1) + vb * 8) = val[u];
            *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o + 2 * W) + vb * 8) = val[u];
            *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, o + 2 * W + 1) + vb * 8) = val[u];
            float v[8];
            unpack8(val[u], v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              os[j] += v[j];
              oq[j] = fmaf(v[j], v[j], oq[j]);
            }
          }
        } else {
          bf16x8 q[U][4];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int pc = pc0 + u * rpi;
            if (pc < p1) {
              const int xc = pc % Wc, yc = pc / Wc;
              const int64_t i0 = (int64_t)(2 * yc) * W + 2 * xc;
              q[u][0] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, i0) + vb * 8);
              q[u][1] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, i0 + 1) + vb * 8);
              q[u][2] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, i0 + W) + vb * 8);
              q[u][3] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(x, f, i0 + W + 1) + vb * 8);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int pc = pc0 + u * rpi;
            if (pc >= p1) break;
            float a[8], b[8], c[8], d[8], r[8];
            unpack8(q[u][0], a);
            unpack8(q[u][1], b);
            unpack8(q[u][2], c);
            unpack8(q[u][3], d);
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = (((a[j] + b[j]) + c[j]) + d[j]) * 0.25f;
            const bf16x8 pk = pack8(r);
            *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, (int64_t)(pc / Wc) * Wc + pc % Wc) + vb * 8) = pk;
            unpack8(pk, r);   // the statistics of what is stored
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              os[j] += r[j];
              oq[j] = fmaf(r[j], r[j], oq[j]);
              is[j] += ((a[j] + b[j]) + c[j]) + d[j];
              iq[j] += ((a[j] * a[j] + b[j] * b[j]) + c[j] * c[j]) + d[j] * d[j];
            }
          }
        }
      }
    }
    if (fits) {
      if (active) {
#pragma unroll
        for (int j = 0; j < 8; ++j) rsm[lane_r * C + vb * 8 + j] = make_float4(os[j], oq[j], is[j], iq[j]);
      }
      __syncthreads();
      if (lane_r == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 t = rsm[vb * 8 + j];
          for (int rr = 1; rr < rpi; ++rr) {
            const float4 u = rsm[rr * C + vb * 8 + j];
            t.x += u.x;
            t.y += u.y;
            t.z += u.z;
            t.w += u.w;
          }
          os[j] = t.x;
          oq[j] = t.y;
          is[j] = t.z;
          iq[j] = t.w;
        }
      }
    }
    if (lane_r == 0) {
      const float k = UP ? 4.f : 1.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (out_part)
          out_part[((int64_t)f * splits + sp) * out_ld + out_c0 + vb * 8 + j] = make_float2(k * os[j], k * oq[j]);
        if (!UP && in_part) in_part[((int64_t)f * splits + sp) * in_ld + vb * 8 + j] = make_float2(is[j], iq[j]);
      }
    }
  }
}

static sf_status launch_resample_gn(int up, sf_view_t x, sf_view_t y, int frames, int H, int W, int C, int splits,
                                    void* out_part, int out_ld, int out_c0, void* in_part, int in_ld,
                                    cudaStream_t st) {
  const int nvec = C / 8;
  const int rpi = nvec <= 256 ? 256 / nvec : 1;
  const size_t smem = nvec <= 256 ? (size_t)rpi * C * sizeof(float4) : 0;
  auto kern = up ? resample_gn_kernel<1> : resample_gn_kernel<0>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_k(kern, dim3((unsigned)splits, (unsigned)frames), dim3(nvec <= 256 ? rpi * nvec : 256), smem, st, x, y, H, W,
           C, splits, (float2*)out_part, out_ld, out_c0, (float2*)in_part, in_ld);
  return launch_status(up ? "sf_upsample2x_gn" : "sf_downsample2x_gn");
}

// ---------------------------------------------------------------------------
// softmax rows: fp32 scores -> bf16 probabilities (kernels.py:272-276)
// ---------------------------------------------------------------------------
template <int PER>
__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* __restrict__ s, int64_t lds,
                                                           bf16* __restrict__ p, int64_t ldp, int n) {
  griddep_wait();
  // PER float4 chunks per thread; n % 4 == 0 and 16-byte aligned rows
  const int64_t row = blockIdx.x;
  const float4* src = reinterpret_cast<const float4*>(s + row * lds);
  const int n4 = n / 4;
  float4 v[PER];
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    v[k] = c < n4 ? src[c] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    m = fmaxf(m, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
  }
  __shared__ float red[8];
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    v[k].x = __expf(v[k].x - m);
    v[k].y = __expf(v[k].y - m);
    v[k].z = __expf(v[k].z - m);
    v[k].w = __expf(v[k].w - m);
    sum += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  sum = warp_sum(sum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float inv = 1.f / tot;
  bf162* dst = reinterpret_cast<bf162*>(p + row * ldp);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int c = threadIdx.x + k * blockDim.x;
    if (c < n4) {
      dst[2 * c] = __floats2bfloat162_rn(v[k].x * inv, v[k].y * inv);
      dst[2 * c + 1] = __floats2bfloat162_rn(v[k].z * inv, v[k].w * inv);
    }
  }
}

// ---------------------------------------------------------------------------
// temporal attention core: one CTA per pixel, T <= 64 tokens of width C.
// S = q k^T * scale (fp32 in smem), softmax, O = P v  (kernels.py:269-308)
// ---------------------------------------------------------------------------
constexpr int TA_MAXT = 64;
constexpr int TA_CHUNK = 32;
__global__ void __launch_bounds__(256) temporal_attn_kernel(sf_view_t qkv, int koff, int voff, sf_view_t out,
                                                            int T, int n_inner, int C, float scale) {
  griddep_wait();
  const int pix = blockIdx.x % n_inner, b = blockIdx.x / n_inner;
  __shared__ float S[TA_MAXT][TA_MAXT + 1];
  __shared__ float qs[TA_MAXT][TA_CHUNK + 1];
  __shared__ float ks[TA_MAXT][TA_CHUNK + 1];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int TT = T * T;
  float acc[TA_MAXT * TA_MAXT / 256];
#pragma unroll
  for (int k = 0; k < TA_MAXT * TA_MAXT / 256; ++k) acc[k] = 0.f;
  for (int c0 = 0; c0 < C; c0 += TA_CHUNK) {
    for (int idx = tid; idx < T * TA_CHUNK; idx += nth) {
      int t = idx / TA_CHUNK, c = idx % TA_CHUNK;
      const bf16* r = row_ptr<const bf16>(qkv, (int64_t)b * T + t, pix);
      bool ok = c0 + c < C;
      qs[t][c] = ok ? __bfloat162float(r[c0 + c]) : 0.f;
      ks[t][c] = ok ? __bfloat162float(r[koff + c0 + c]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TA_MAXT * TA_MAXT / 256; ++k) {
      int e = tid + k * 256;
      if (e < TT) {
        int i = e / T, j = e % T;
        float a = 0.f;
#pragma unroll 8
        for (int c = 0; c < TA_CHUNK; ++c) a += qs[i][c] * ks[j][c];
        acc[k] += a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < TA_MAXT * TA_MAXT / 256; ++k) {
    int e = tid + k * 256;
    if (e < TT) S[e / T][e % T] = acc[k] * scale;
  }
  __syncthreads();
  // softmax: one warp per row
  const int warp = tid >> 5, lane = tid & 31;
  for (int i = warp; i < T; i += nth / 32) {
    float a = lane < T ? S[i][lane] : -INFINITY;
    float bb = lane + 32 < T ? S[i][lane + 32] : -INFINITY;
    float m = warp_max(fmaxf(a, bb));
    a = lane < T ? __expf(a - m) : 0.f;
    bb = lane + 32 < T ? __expf(bb - m) : 0.f;
    float inv = 1.f / warp_sum(a + bb);
    if (lane < T) S[i][lane] = a * inv;
    if (lane + 32 < T) S[i][lane + 32] = bb * inv;
  }
  __syncthreads();
  // O = P v, chunked over channels (reuse qs as the v chunk)
  for (int c0 = 0; c0 < C; c0 += TA_CHUNK) {
    for (int idx = tid; idx < T * TA_CHUNK; idx += nth) {
      int t = idx / TA_CHUNK, c = idx % TA_CHUNK;
      const bf16* r = row_ptr<const bf16>(qkv, (int64_t)b * T + t, pix);
      qs[t][c] = c0 + c < C ? __bfloat162float(r[voff + c0 + c]) : 0.f;
    }
    __syncthreads();
    for (int idx = tid; idx < T * TA_CHUNK; idx += nth) {
      int t = idx / TA_CHUNK, c = idx % TA_CHUNK;
      if (c0 + c < C) {
        float a = 0.f;
        for (int j = 0; j < T; ++j) a += S[t][j] * qs[j][c];
        row_ptr<bf16>(out, (int64_t)b * T + t, pix)[c0 + c] = __float2bfloat16(a);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// temporal attention core, tensor-core version for T <= 32: one warp per pixel.
// S (32x32, fp32 fragments) accumulated over 64-channel chunks with
// mma.sync m16n8k16; softmax on the fragments (quad shuffles); P re-packed as
// the A operand; O = P V per 64-channel chunk, V read with ldmatrix.trans.
// Rows t >= T are zero-filled and their scores masked.
// ---------------------------------------------------------------------------
constexpr int TQ_WARPS = 4, TQ_CH = 64, TQ_LD = TQ_CH + 8;

__device__ __forceinline__ void tq_ldsm_x4(unsigned* r, const void* p) {
  unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(s));
}
__device__ __forceinline__ void tq_ldsm_x4_t(unsigned* r, const void* p) {
  unsigned s = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(s));
}
__device__ __forceinline__ void tq_mma(float* c, const unsigned* a, unsigned b0, unsigned b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ unsigned pack_bf2(float a, float b) {
  bf162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<unsigned*>(&h);
}

// ---------------------------------------------------------------------------
// GroupNorm-apply + SiLU fused into a narrow projection (the network's out_norm -> out_conv,
// kernels.py:228-253 then 181-201 regrouped per tap: Y[p][n] = sum_c SiLU(GN(x))[p][c] W[n][c],
// n = tap * cout + co).  The normalised activations never reach HBM: each warp loads 16 rows of x,
// applies y = SiLU(x * ss + bb) (ss = rstd * gamma, bb = beta - mean * ss: gn_apply_kernel's exact
// arithmetic, rounded to bf16 as that kernel stores it) into its shared-memory A tile, and multiplies
// it with the resident W (bf16 [48][C]) on mma.sync m16n8k16; fp32 out.  Each element is
// transformed once (the per-tap projection reads every pixel once, unlike a 3x3 implicit GEMM).
// ---------------------------------------------------------------------------
constexpr int GP_WARPS = 16, GP_NP = 48;   // output columns padded to 6 n-tiles of 8
constexpr int GP_LDA = 64 + 8;              // one 64-channel K chunk per A buffer, +16 B per row
__global__ void __launch_bounds__(GP_WARPS * 32) gn_project_kernel(
    sf_view_t x, int frames, int n_inner, int C, int groups, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ gamma, const float* __restrict__ beta, int act,
    const bf16* __restrict__ w, int N, float* __restrict__ out, int64_t ldo) {
  griddep_wait();
  extern __shared__ __align__(16) uint8_t gp_raw[];
  const int LD = C + 8;   // +16 B per row: conflict-free ldmatrix
  bf16* sW = reinterpret_cast<bf16*>(gp_raw);                        // [GP_NP][LD]
  bf16* sA = sW + GP_NP * LD;                                        // [GP_WARPS][2][16][GP_LDA]
  float2* sT = reinterpret_cast<float2*>(sA + GP_WARPS * 2 * 16 * GP_LDA);   // [GP_WARPS][2][C] (scale, shift)
  for (int i = threadIdx.x; i < GP_NP * (C / 8); i += blockDim.x) {
    const int n = i / (C / 8), v = i % (C / 8);
    *reinterpret_cast<bf16x8*>(sW + n * LD + v * 8) =
        n < N ? *reinterpret_cast<const bf16x8*>(w + (int64_t)n * C + v * 8) : bf16x8{make_uint4(0, 0, 0, 0)};
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bf16* abuf = sA + warp * 2 * 16 * GP_LDA;
  float2* tab = sT + warp * 2 * C;
  const int cg = C / groups, nk = C / 64;
  const int64_t rows = (int64_t)frames * n_inner;
  // blocks take contiguous shares of the 16-row tiles (a block touches one or two frames)
  const int64_t ntiles = (rows + 15) / 16;
  const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
  // a K chunk = 16 rows x 8 vectors: lane -> rows lane / 8 + {0, 4, 8, 12}, vector lane % 8
  const int lr = lane >> 3, lv = lane & 7;
  int fa = -1, fb = -1;
  for (int64_t t = t0 + warp; t < t1; t += GP_WARPS) {
    const int64_t r0 = t * 16;
    const int f0 = (int)(r0 / n_inner), f1 = (int)(min(r0 + 15, rows - 1) / n_inner);
    if (f0 != fa || f1 != fb) {
      // y = x * ss + bb, ss = rstd * gamma, bb = beta - mean * ss (gn_apply_kernel's arithmetic), per
      // channel of the tile's first / last frame (a 16-row tile spans at most two frames: n_inner >= 16)
      for (int c = lane; c < C; c += 32) {
        const int g = c / cg;
        const float s0 = __ldg(rstd + f0 * groups + g) * __ldg(gamma + c);
        const float s1 = __ldg(rstd + f1 * groups + g) * __ldg(gamma + c);
        tab[c] = make_float2(s0, fmaf(-__ldg(mean + f0 * groups + g), s0, __ldg(beta + c)));
        tab[C + c] = make_float2(s1, fmaf(-__ldg(mean + f1 * groups + g), s1, __ldg(beta + c)));
      }
      fa = f0;
      fb = f1;
      __syncwarp();
    }
    // row -> (frame, local row) without divisions: rows from `split` on belong to frame f0 + 1
    const int split = (int)min((int64_t)16, (int64_t)(f0 + 1) * n_inner - r0);
    const int64_t base0 = r0 - (int64_t)f0 * n_inner;
    const int nvalid = (int)min((int64_t)16, rows - r0);
    const bf16* src[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rr = lr + 4 * u;
      const bool second = rr >= split;
      src[u] = rr < nvalid ? row_ptr<const bf16>(x, f0 + (second ? 1 : 0), second ? rr - split : base0 + rr) + lv * 8
                           : nullptr;
    }
    bf16x8 cur[4], nxt[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (src[u]) cur[u] = *reinterpret_cast<const bf16x8*>(src[u]);
    float acc[GP_NP / 8][4];
#pragma unroll
    for (int j = 0; j < GP_NP / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    for (int kc = 0; kc < nk; ++kc) {
      if (kc + 1 < nk) {   // the next chunk's loads fly while this one is transformed and multiplied
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (src[u]) nxt[u] = *reinterpret_cast<const bf16x8*>(src[u] + (kc + 1) * 64);
      }
      bf16* a = abuf + (kc & 1) * 16 * GP_LDA;
      // this lane's 8 channels' (ss, bb) once per chunk (its 4 rows share them unless the tile
      // straddles two frames)
      float4 sbA[4];
      {
        const float4* tv = reinterpret_cast<const float4*>(tab + kc * 64 + lv * 8);
#pragma unroll
        for (int q = 0; q < 4; ++q) sbA[q] = tv[q];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = lr + 4 * u;
        float fv[8];
        if (src[u]) {
          float4 sb4[4];
          if (rr >= split) {
            const float4* tv = reinterpret_cast<const float4*>(tab + C + kc * 64 + lv * 8);
#pragma unroll
            for (int q = 0; q < 4; ++q) sb4[q] = tv[q];
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) sb4[q] = sbA[q];
          }
          unpack8(cur[u], fv);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 sb = sb4[q];   // (ss, bb) of channels 2q, 2q+1
            const float ta = fmaf(fv[2 * q], sb.x, sb.y), tb = fmaf(fv[2 * q + 1], sb.z, sb.w);
            fv[2 * q] = act ? silu_f(ta) : ta;
            fv[2 * q + 1] = act ? silu_f(tb) : tb;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) fv[j] = 0.f;
        }
        *reinterpret_cast<bf16x8*>(a + rr * GP_LDA + lv * 8) = pack8(fv);
      }
      __syncwarp();
#pragma unroll
      for (int kk = 0; kk < 64; kk += 16) {
        unsigned af[4];
        tq_ldsm_x4(af, a + (lane & 15) * GP_LDA + kk + (lane >> 4) * 8);
#pragma unroll
        for (int j = 0; j < GP_NP / 8; j += 2) {
          unsigned b[4];
          const int nrow = j * 8 + (lane & 7) + ((lane >> 4) << 3);
          tq_ldsm_x4(b, sW + nrow * LD + kc * 64 + kk + ((lane >> 3) & 1) * 8);
          tq_mma(acc[j], af, b[0], b[1]);
          tq_mma(acc[j + 1], af, b[2], b[3]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
    }
    const int64_t ra = r0 + (lane >> 2), rb = ra + 8;
#pragma unroll
    for (int j = 0; j < GP_NP / 8; ++j) {
      const int c = j * 8 + (lane & 3) * 2;
      if (c < N) {   // N even: the pair (c, c + 1) is in range together
        if (ra < rows) *reinterpret_cast<float2*>(out + ra * ldo + c) = make_float2(acc[j][0], acc[j][1]);
        if (rb < rows) *reinterpret_cast<float2*>(out + rb * ldo + c) = make_float2(acc[j][2], acc[j][3]);
      }
    }
    __syncwarp();   // the A buffers are rewritten by the next tile
  }
}

sf_status gn_project_launch(sf_view_t x, int frames, int n_inner, int C, int groups, const float* mean,
                            const float* rstd, const float* gamma, const float* beta, int act, const void* w, int N,
                            float* out, int64_t ldo, cudaStream_t st) {
  const size_t smem = ((size_t)GP_NP * (C + 8) + (size_t)GP_WARPS * 2 * 16 * GP_LDA) * sizeof(bf16) +
                      (size_t)GP_WARPS * 2 * C * sizeof(float2);
  static size_t set = 48 * 1024;
  if (smem > set) {
    cudaFuncSetAttribute(gn_project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set = smem;
  }
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gn_project_kernel, GP_WARPS * 32, smem);
    if (occ < 1) occ = 1;
  }
  const int64_t tiles = ((int64_t)frames * n_inner + 15) / 16;
  int64_t grid = (int64_t)num_sms() * occ;
  const int64_t most = (tiles + GP_WARPS - 1) / GP_WARPS;
  if (grid > most) grid = most;
  launch_k(gn_project_kernel, dim3((unsigned)grid), dim3(GP_WARPS * 32), smem, st, x, frames, n_inner, C, groups, mean,
           rstd, gamma, beta, act, (const bf16*)w, N, out, ldo);
  return launch_status("sf_group_norm_project");
}

// copy a [32 tokens][64 ch] chunk (columns col0..col0+63) into smem, zero rows t >= T / ch >= C
__device__ __forceinline__ void tq_load(bf16 (*dst)[TQ_LD], const sf_view_t& v, int b, int T, int pix, int col0,
                                        int cvalid, int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int idx = lane + 32 * k;     // 256 vectors = 32 rows x 8
    int t = idx >> 3, c = (idx & 7) * 8;
    bf16x8 val;
    if (t < T && c < cvalid) {
      val = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(v, (int64_t)b * T + t, pix) + col0 + c);
    } else {
      val.u = make_uint4(0u, 0u, 0u, 0u);
    }
    *reinterpret_cast<bf16x8*>(&dst[t][c]) = val;
  }
}

// register-staged variant: issue a chunk's loads early (tq_fetch), store them to smem later (tq_put),
// so the next chunk is in flight while the current one is in the MMAs
struct TqChunk {
  bf16x8 v[8];
};
__device__ __forceinline__ void tq_fetch(TqChunk& r, const sf_view_t& v, int b, int T, int pix, int col0, int cvalid,
                                         int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int idx = lane + 32 * k, t = idx >> 3, c = (idx & 7) * 8;
    if (t < T && c < cvalid)
      r.v[k] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(v, (int64_t)b * T + t, pix) + col0 + c);
    else
      r.v[k].u = make_uint4(0u, 0u, 0u, 0u);
  }
}
__device__ __forceinline__ void tq_put(bf16 (*dst)[TQ_LD], const TqChunk& r, int lane) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int idx = lane + 32 * k;
    *reinterpret_cast<bf16x8*>(&dst[idx >> 3][(idx & 7) * 8]) = r.v[k];
  }
}

#ifndef TQ_MINB
#define TQ_MINB 1   // resident blocks per SM the register allocation must allow (tuning: -DTQ_MINB=n)
#endif
#ifndef TQ_SPLIT_MINB
#define TQ_SPLIT_MINB 1   // the same for the channel-split variant (tuning: -DTQ_SPLIT_MINB=n)
#endif
// SPLIT = 1: one warp per pixel.  SPLIT = TQ_WARPS: the block's warps share one pixel (few-pixel deep
// levels, e.g. 576 / 144 pixels, where one warp per pixel leaves most SMs idle): warp w takes the
// channel chunks w, w + SPLIT, ...; the partial scores are summed across warps in shared memory in a
// fixed order (deterministic), every warp runs the (cheap) softmax, and each writes its own chunks of O.
template <int SPLIT>
__global__ void __launch_bounds__(TQ_WARPS * 32, SPLIT > 1 ? TQ_SPLIT_MINB : TQ_MINB) temporal_attn_mma_kernel(sf_view_t qkv, int koff, int voff,
                                                                          sf_view_t out, int B, int T, int n_inner,
                                                                          int C, float scale_log2) {
  griddep_wait();
  extern __shared__ __align__(16) unsigned char tq_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bf16 (*qs)[TQ_LD] = reinterpret_cast<bf16 (*)[TQ_LD]>(tq_smem + warp * 3 * 32 * TQ_LD * 2);
  bf16 (*ks)[TQ_LD] = qs + 32;
  bf16 (*vs)[TQ_LD] = qs + 64;
  const int64_t gp = SPLIT == 1 ? (int64_t)blockIdx.x * TQ_WARPS + warp : (int64_t)blockIdx.x;  // (b, pix)
  if (gp >= (int64_t)B * n_inner) return;
  const int cs = SPLIT == 1 ? 0 : warp * TQ_CH;   // this warp's first channel chunk
  constexpr int CSTEP = SPLIT * TQ_CH;
  const int b = gp / n_inner, pix = gp % n_inner;
  float sacc[2][4][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) sacc[i][j][e] = 0.f;
  TqChunk rq, rk;
  if (SPLIT == 1 || cs < C) {
    tq_fetch(rq, qkv, b, T, pix, cs, min(TQ_CH, C - cs), lane);
    tq_fetch(rk, qkv, b, T, pix, koff + cs, min(TQ_CH, C - cs), lane);
  }
  for (int c0 = cs; c0 < C; c0 += CSTEP) {
    tq_put(qs, rq, lane);
    tq_put(ks, rk, lane);
    __syncwarp();
    if (c0 + CSTEP < C) {
      const int nv = min(TQ_CH, C - c0 - CSTEP);
      tq_fetch(rq, qkv, b, T, pix, c0 + CSTEP, nv, lane);
      tq_fetch(rk, qkv, b, T, pix, koff + c0 + CSTEP, nv, lane);
    }
#pragma unroll
    for (int kk = 0; kk < TQ_CH; kk += 16) {
      unsigned a[2][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) tq_ldsm_x4(a[mi], &qs[mi * 16 + (lane & 15)][kk + (lane >> 4) * 8]);
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        unsigned r[4];
        tq_ldsm_x4(r, &ks[nj * 16 + (lane & 7) + ((lane >> 4) << 3)][kk + ((lane >> 3) & 1) * 8]);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          tq_mma(sacc[mi][2 * nj], a[mi], r[0], r[1]);
          tq_mma(sacc[mi][2 * nj + 1], a[mi], r[2], r[3]);
        }
      }
    }
    __syncwarp();
  }
  if constexpr (SPLIT > 1) {
    // sum the warps' partial scores (fragment layout, fixed warp order) through shared memory
    float* red = reinterpret_cast<float*>(tq_smem);
    constexpr int PER = 2 * 4 * 4 * 32;   // floats per warp
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) red[warp * PER + ((i * 4 + j) * 4 + e) * 32 + lane] = sacc[i][j][e];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < SPLIT; ++w) v += red[w * PER + ((i * 4 + j) * 4 + e) * 32 + lane];
          sacc[i][j][e] = v;
        }
    __syncthreads();
  }
  // softmax over columns (keys) per row; lane holds rows lane/4 (+8) of each m-tile
  float rsum[2][2];
  const int colq = (lane & 3) * 2;
#pragma unroll
  for (int mi = 0; mi < 2; ++mi) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float m = -INFINITY;
#pragma unroll
      for (int nj = 0; nj < 4; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int col = nj * 8 + colq + e;
          float v = col < T ? sacc[mi][nj][h * 2 + e] * scale_log2 : -INFINITY;
          sacc[mi][nj][h * 2 + e] = v;
          m = fmaxf(m, v);
        }
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      float sum = 0.f;
#pragma unroll
      for (int nj = 0; nj < 4; ++nj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float pv = exp2f(sacc[mi][nj][h * 2 + e] - m);
          sacc[mi][nj][h * 2 + e] = pv;
          sum += pv;
        }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      rsum[mi][h] = 1.f / sum;
    }
  }
  // P as A fragments: k-step kk covers keys 16kk..16kk+15 = n-tiles 2kk, 2kk+1
  unsigned pa[2][2][4];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      pa[mi][kk][0] = pack_bf2(sacc[mi][2 * kk][0], sacc[mi][2 * kk][1]);
      pa[mi][kk][1] = pack_bf2(sacc[mi][2 * kk][2], sacc[mi][2 * kk][3]);
      pa[mi][kk][2] = pack_bf2(sacc[mi][2 * kk + 1][0], sacc[mi][2 * kk + 1][1]);
      pa[mi][kk][3] = pack_bf2(sacc[mi][2 * kk + 1][2], sacc[mi][2 * kk + 1][3]);
    }
  TqChunk rv;
  if (SPLIT == 1 || cs < C) tq_fetch(rv, qkv, b, T, pix, voff + cs, min(TQ_CH, C - cs), lane);
  for (int c0 = cs; c0 < C; c0 += CSTEP) {
    const int cv = min(TQ_CH, C - c0);
    tq_put(vs, rv, lane);
    __syncwarp();
    if (c0 + CSTEP < C) tq_fetch(rv, qkv, b, T, pix, voff + c0 + CSTEP, min(TQ_CH, C - c0 - CSTEP), lane);
    float oacc[2][8][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) oacc[i][j][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
      for (int nj = 0; nj < 4; ++nj) {
        unsigned r[4];
        // V [k=token][n=ch]: trans loads (k0-7,n),(k8-15,n),(k0-7,n+8),(k8-15,n+8)
        tq_ldsm_x4_t(r, &vs[kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8][nj * 16 + (lane >> 4) * 8]);
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          tq_mma(oacc[mi][2 * nj], pa[mi][kk], r[0], r[1]);
          tq_mma(oacc[mi][2 * nj + 1], pa[mi][kk], r[2], r[3]);
        }
      }
    }
    // O chunk -> smem (the q tile is free) -> 16-byte row stores
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = mi * 16 + (lane >> 2) + h * 8;
#pragma unroll
        for (int nj = 0; nj < 8; ++nj)
          *reinterpret_cast<unsigned*>(&qs[t][nj * 8 + colq]) =
              pack_bf2(oacc[mi][nj][h * 2] * rsum[mi][h], oacc[mi][nj][h * 2 + 1] * rsum[mi][h]);
      }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = lane + 32 * k, t = idx >> 3, c = (idx & 7) * 8;
      if (t < T && c < cv)
        *reinterpret_cast<bf16x8*>(row_ptr<bf16>(out, (int64_t)b * T + t, pix) + c0 + c) =
            *reinterpret_cast<const bf16x8*>(&qs[t][c]);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// latent-edge convolutions with tiny channel counts (in_conv / out_conv)
// ---------------------------------------------------------------------------
// in_conv: tiny cin, fp32 input.  A warp covers 32 consecutive pixels for one
// chunk of 32 output channels; the [9][cin][cout] weights sit in shared memory
// and every weight read is a warp-wide broadcast.
constexpr int SC_THREADS = 128;
template <int SC_CO>
__global__ void __launch_bounds__(SC_THREADS) conv_smallcin_kernel(const float* __restrict__ x, int frames, int H,
                                                                   int W, int cin, const float* __restrict__ wt,
                                                                   const float* __restrict__ bias, int cout,
                                                                   sf_view_t y) {
  griddep_wait();
  extern __shared__ float wsm[];  // [9][cin][cout]
  const int nw = 9 * cin * cout;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) wsm[i] = wt[i];
  __syncthreads();
  const int nchunk = cout / SC_CO;
  const int64_t npix = (int64_t)frames * H * W;
  const int64_t total = npix * nchunk;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // idx -> (chunk, pixel) with pixels fastest so a warp shares one weight chunk
    const int64_t p = idx % npix;
    const int ch = (int)(idx / npix);
    const int px = p % W, py = (p / W) % H, f = p / ((int64_t)W * H);
    float acc[SC_CO];
#pragma unroll
    for (int j = 0; j < SC_CO; ++j) acc[j] = bias[ch * SC_CO + j];
    for (int tap = 0; tap < 9; ++tap) {
      const int yy = py + tap / 3 - 1, xx = px + tap % 3 - 1;
      const bool ok = yy >= 0 && yy < H && xx >= 0 && xx < W;
      const float* src = x + (((int64_t)f * H + yy) * W + xx) * cin;
      for (int ci = 0; ci < cin; ++ci) {
        const float a = ok ? __ldg(src + ci) : 0.f;
        const float4* wr = reinterpret_cast<const float4*>(wsm + ((tap * cin + ci) * cout + ch * SC_CO));
#pragma unroll
        for (int j = 0; j < SC_CO / 4; ++j) {
          const float4 w4 = wr[j];
          acc[4 * j] += a * w4.x;
          acc[4 * j + 1] += a * w4.y;
          acc[4 * j + 2] += a * w4.z;
          acc[4 * j + 3] += a * w4.w;
        }
      }
    }
    bf16* dst = row_ptr<bf16>(y, f, (int64_t)py * W + px) + ch * SC_CO;
#pragma unroll
    for (int j = 0; j < SC_CO / 8; ++j) reinterpret_cast<bf16x8*>(dst)[j] = pack8(acc + 8 * j);
  }
}

// 3x3 conv with few input channels (the UNet in_conv: latent cin = 4 -> 320)
// as a tensor-core implicit GEMM: K = 9*cin taps padded to 16, mma.sync bf16.
// Each CTA gathers the im2col tile of 128 pixels straight from the fp32
// latent into shared memory (taps outside the image are zero), keeps the whole
// weight matrix [cout][K] resident, and writes bf16 output through a staging
// tile so every row leaves as full 128-byte segments.
constexpr int SCM_THREADS = 256, SCM_WARPS = SCM_THREADS / 32, SCM_NCH = 64;
template <int KP>
struct ScmLayout {
  static constexpr int LDA = KP + 8;                 // +16 B per row: conflict-free ldmatrix
  static constexpr int LDO = SCM_NCH + 8;
  static constexpr int A_ELEMS = SCM_WARPS * 16 * LDA;   // per warp: its 16-pixel im2col tile
  static constexpr int O_ELEMS = SCM_WARPS * 16 * LDO;   // per warp: a 16 x 64 output staging tile
};
// The network's in_conv (kernels.py:181-201 with 4 input channels): im2col rows of K = 9 * cin
// (padded to KP) gathered from the fp32 latent, multiplied on mma.sync by the resident weights.
// Every warp works on its own tasks -- task = (frame, split): a contiguous run of 16-pixel tiles of
// one frame -- with warp-private im2col / staging tiles, so no block barrier follows the weight load.
// With part != nullptr the warp also sums the bf16 values it stores per channel over its task and
// writes part[(frame * splits + split) * cout + c] (float2 sum, sum sq): the statistics of the
// GroupNorm that reads this output (unet.py:213-216, in_conv -> down_blocks.0.res.norm1).
template <int KP>
__global__ void __launch_bounds__(SCM_THREADS) conv_smallcin_mma_kernel(const float* __restrict__ x, int frames, int H,
                                                                       int W, int cin, const float* __restrict__ wt,
                                                                       const float* __restrict__ bias, int cout,
                                                                       sf_view_t y, int splits, float2* part) {
  griddep_wait();
  using L = ScmLayout<KP>;
  extern __shared__ __align__(16) uint8_t scm_raw[];
  bf16* sA0 = reinterpret_cast<bf16*>(scm_raw);
  bf16* sO0 = sA0 + L::A_ELEMS;
  bf16* sB = sO0 + L::O_ELEMS;  // [cout][LDA]
  float* sBias = reinterpret_cast<float*>(sB + (size_t)cout * L::LDA);
  const int K = 9 * cin;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bf16* sA = sA0 + warp * 16 * L::LDA;
  bf16* sO = sO0 + warp * 16 * L::LDO;
  float2* sP = reinterpret_cast<float2*>(sBias + cout) + (size_t)warp * cout;   // [cout] task sums (part != 0)
  // weights [9][cin][cout] fp32 -> [cout][k = tap*cin + ci] bf16, zero past K
  for (int i = threadIdx.x; i < cout * KP; i += SCM_THREADS) {
    const int co = i / KP, k = i % KP;
    sB[co * L::LDA + k] = __float2bfloat16(k < K ? wt[(size_t)k * cout + co] : 0.f);
  }
  for (int i = threadIdx.x; i < cout; i += SCM_THREADS) sBias[i] = bias[i];
  // K padding columns of the im2col tiles stay zero for every tile
  for (int i = lane; i < 16 * (KP - K); i += 32) sA[(i / (KP - K)) * L::LDA + K + i % (KP - K)] = __float2bfloat16(0.f);
  __syncthreads();
  const int HW = H * W;
  const int tpf = (HW + 15) / 16;                  // 16-pixel tiles per frame (none straddles frames)
  const int tps = (tpf + splits - 1) / splits;     // tiles per split
  const int64_t ntasks = (int64_t)frames * splits;
  const int nch = cout / SCM_NCH;
  for (int64_t task = (int64_t)blockIdx.x * SCM_WARPS + warp; task < ntasks; task += (int64_t)gridDim.x * SCM_WARPS) {
    const int f = (int)(task / splits), sp = (int)(task % splits);
    const int ta = sp * tps, tb = min(tpf, ta + tps);
    if (part != nullptr)   // lane-owned columns 2 lane, 2 lane + 1 of every 64-channel chunk
      for (int c = 2 * lane; c < cout; c += 64) sP[c] = sP[c + 1] = make_float2(0.f, 0.f);
    for (int t = ta; t < tb; ++t) {
      const int q0 = t * 16;
      // im2col: one (pixel, tap) per lane iteration, cin consecutive floats
      for (int i = lane; i < 16 * 9; i += 32) {
        const int r = i / 9, tap = i - r * 9;
        const int pix = q0 + r;
        bf16* dst = sA + r * L::LDA + tap * cin;
        const float* src = nullptr;
        if (pix < HW) {
          const int py = pix / W, px = pix - py * W;
          const int yy = py + tap / 3 - 1, xx = px + tap % 3 - 1;
          if (yy >= 0 && yy < H && xx >= 0 && xx < W) src = x + ((int64_t)f * HW + (int64_t)yy * W + xx) * cin;
        }
        if (cin == 4) {
          float4 v = src ? __ldg(reinterpret_cast<const float4*>(src)) : make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<unsigned*>(dst) = pack_bf2(v.x, v.y);
          *reinterpret_cast<unsigned*>(dst + 2) = pack_bf2(v.z, v.w);
        } else {
          for (int ci = 0; ci < cin; ++ci) dst[ci] = __float2bfloat16(src ? __ldg(src + ci) : 0.f);
        }
      }
      __syncwarp();
      unsigned af[KP / 16][4];
#pragma unroll
      for (int kk = 0; kk < KP / 16; ++kk) tq_ldsm_x4(af[kk], sA + (lane & 15) * L::LDA + kk * 16 + (lane >> 4) * 8);
      const int nvalid = min(16, HW - q0);
      for (int ch = 0; ch < nch; ++ch) {
        const int n0 = ch * SCM_NCH;
        float acc[SCM_NCH / 8][4];
#pragma unroll
        for (int j = 0; j < SCM_NCH / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KP / 16; ++kk) {
#pragma unroll
          for (int j = 0; j < SCM_NCH / 8; j += 2) {
            unsigned b[4];
            const int nrow = n0 + j * 8 + (lane & 7) + ((lane >> 4) << 3);
            tq_ldsm_x4(b, sB + nrow * L::LDA + kk * 16 + ((lane >> 3) & 1) * 8);
            tq_mma(acc[j], af[kk], b[0], b[1]);
            tq_mma(acc[j + 1], af[kk], b[2], b[3]);
          }
        }
        // bias, bf16, the warp's 16 x 64 staging tile
        const int r0 = lane >> 2;
#pragma unroll
        for (int j = 0; j < SCM_NCH / 8; ++j) {
          const int c = j * 8 + (lane & 3) * 2;
          const float b0 = sBias[n0 + c], b1 = sBias[n0 + c + 1];
          *reinterpret_cast<unsigned*>(sO + r0 * L::LDO + c) = pack_bf2(acc[j][0] + b0, acc[j][1] + b1);
          *reinterpret_cast<unsigned*>(sO + (r0 + 8) * L::LDO + c) = pack_bf2(acc[j][2] + b0, acc[j][3] + b1);
        }
        __syncwarp();
        // 16 rows x 128 B: 8 lanes per row, 16 B each, 4 rows per pass
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = k * 4 + (lane >> 3), v = lane & 7;
          if (r < nvalid)
            *reinterpret_cast<bf16x8*>(row_ptr<bf16>(y, f, q0 + r) + n0 + v * 8) =
                *reinterpret_cast<const bf16x8*>(sO + r * L::LDO + v * 8);
        }
        if (part != nullptr) {
          // the stored values' sums: lane owns columns 2 lane, 2 lane + 1 of the chunk, rows in order
          // four independent row chains (rows r = 4i + u), combined (0+1)+(2+3) per tile
          float4 acc4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) acc4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int r4 = 0; r4 < 16; r4 += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (r4 + u < nvalid) {
                const float2 v2 =
                    __bfloat1622float2(*reinterpret_cast<const bf162*>(sO + (r4 + u) * L::LDO + 2 * lane));
                acc4[u].x += v2.x;
                acc4[u].y = fmaf(v2.x, v2.x, acc4[u].y);
                acc4[u].z += v2.y;
                acc4[u].w = fmaf(v2.y, v2.y, acc4[u].w);
              }
            }
          }
          float2 a = sP[n0 + 2 * lane], b = sP[n0 + 2 * lane + 1];
          a.x += (acc4[0].x + acc4[1].x) + (acc4[2].x + acc4[3].x);
          a.y += (acc4[0].y + acc4[1].y) + (acc4[2].y + acc4[3].y);
          b.x += (acc4[0].z + acc4[1].z) + (acc4[2].z + acc4[3].z);
          b.y += (acc4[0].w + acc4[1].w) + (acc4[2].w + acc4[3].w);
          sP[n0 + 2 * lane] = a;
          sP[n0 + 2 * lane + 1] = b;
        }
        __syncwarp();
      }
    }
    if (part != nullptr) {
      float2* dst = part + ((int64_t)f * splits + sp) * cout;
      for (int c = 2 * lane; c < cout; c += 64) {
        dst[c] = sP[c];
        dst[c + 1] = sP[c + 1];
      }
    }
  }
}

template <int KP>
static sf_status conv_smallcin_mma_launch(const float* x, int frames, int H, int W, int cin, const float* w,
                                          const float* bias, int cout, sf_view_t y, int splits, void* part,
                                          cudaStream_t st) {
  using L = ScmLayout<KP>;
  // the per-warp sums (sP) only when partials are requested: without them three blocks fit per SM
  const size_t smem = (size_t)(L::A_ELEMS + L::O_ELEMS + cout * L::LDA) * sizeof(bf16) + cout * sizeof(float) +
                      (part ? (size_t)SCM_WARPS * cout * sizeof(float2) : 0);
  static size_t cfg = 0;
  if (smem > 48 * 1024 && smem > cfg) {
    cudaFuncSetAttribute(conv_smallcin_mma_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cfg = smem;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_smallcin_mma_kernel<KP>, SCM_THREADS, smem);
  // without partials the split count only shapes the work: ~2 tasks per warp slot
  const int tpf = (H * W + 15) / 16;
  if (!part) splits = std::max(1, std::min(tpf, (2 * num_sms() * std::max(per_sm, 1) * SCM_WARPS + frames - 1) / frames));
  const int64_t ntasks = (int64_t)frames * splits;
  const int64_t grid = std::min<int64_t>((ntasks + SCM_WARPS - 1) / SCM_WARPS, (int64_t)num_sms() * std::max(per_sm, 1));
  launch_k(conv_smallcin_mma_kernel<KP>, dim3((unsigned)grid), dim3(SCM_THREADS), smem, st, x, frames, H, W, cin, w,
           bias, cout, y, splits, (float2*)part);
  return launch_status("sf_conv3x3_smallcin(mma)");
}

// out_conv (cout < 16) as "project then shift-and-sum": y = per-tap projections
// [f][p][tap*cout + co] from one plain GEMM; each output sums its 9 shifted taps.
__global__ void conv_tapsum_kernel(const float* __restrict__ y, int ldy, int frames, int H, int W, int cout,
                                   const float* __restrict__ bias, sf_view_t out) {
  griddep_wait();
  const int HW = H * W;
  const int64_t total = (int64_t)frames * HW * cout;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int co = (int)(idx % cout);
    const int64_t pp = idx / cout;
    const int f = (int)(pp / HW), pix = (int)(pp - (int64_t)f * HW);
    const int py = pix / W, px = pix - py * W;
    float acc = bias ? __ldg(bias + co) : 0.f;
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int yy = py + tap / 3 - 1, xx = px + tap % 3 - 1;
      if (yy >= 0 && yy < H && xx >= 0 && xx < W)
        acc += __ldg(y + ((int64_t)f * HW + (int64_t)yy * W + xx) * ldy + tap * cout + co);
    }
    row_ptr<float>(out, f, pix)[co] = acc;
  }
}

__global__ void gemv_kernel(const float* __restrict__ Wm, const float* __restrict__ e, const float* __restrict__ b,
                            float* __restrict__ y, int N, int K) {
  griddep_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= N) return;
  float a = 0.f;
  for (int k = lane; k < K; k += 32) a += Wm[(int64_t)warp * K + k] * e[k];
  a = warp_sum(a);
  if (lane == 0) y[warp] = a + (b ? b[warp] : 0.f);
}

__global__ void transpose_f32_kernel(const float* __restrict__ x, float* __restrict__ y, int frames, int A, int B,
                                     int to_rows) {
  griddep_wait();
  // to_rows: x[f][A=C][B=HW] -> y[f][HW][C];  else x[f][A=HW][B=C] -> y[f][C][HW]
  const int64_t total = (int64_t)frames * A * B;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t f = idx / ((int64_t)A * B);
    int r = idx % ((int64_t)A * B);
    int a = r / B, bb = r % B;
    y[f * A * B + (int64_t)bb * A + a] = x[idx];
  }
}

__global__ void axpy_kernel(float* __restrict__ x, const float* __restrict__ e, float alpha, int64_t n) {
  griddep_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = x[i] - alpha * e[i];
}

// ---------------------------------------------------------------------------
// similarity: fixed-order fp64 partials, then one block combines
// ---------------------------------------------------------------------------
constexpr int DOT_BLOCKS = 592, DOT_THREADS = 256;

__global__ void dot3_partial_kernel(const bf16* __restrict__ a, const bf16* __restrict__ b, int64_t n,
                                    double* __restrict__ part) {
  griddep_wait();
  double aa = 0, bb = 0, ab = 0;
  const int64_t nv = n / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float fa[8], fb[8];
    unpack8(reinterpret_cast<const bf16x8*>(a)[i], fa);
    unpack8(reinterpret_cast<const bf16x8*>(b)[i], fb);
    float sa = 0, sb = 0, sab = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sa += fa[j] * fa[j];
      sb += fb[j] * fb[j];
      sab += fa[j] * fb[j];
    }
    aa += sa;
    bb += sb;
    ab += sab;
  }
  for (int64_t i = nv * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = __bfloat162float(a[i]), y = __bfloat162float(b[i]);
    aa += x * x;
    bb += y * y;
    ab += x * y;
  }
  __shared__ double red[3][DOT_THREADS / 32];
  aa = warp_sum_d(aa);
  bb = warp_sum_d(bb);
  ab = warp_sum_d(ab);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = aa;
    red[1][threadIdx.x >> 5] = bb;
    red[2][threadIdx.x >> 5] = ab;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0;
    for (int w = 0; w < DOT_THREADS / 32; ++w) s += red[threadIdx.x][w];
    part[blockIdx.x * 3 + threadIdx.x] = s;
  }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int nparts, int width, double* __restrict__ out) {
  griddep_wait();
  // out[j] = sum_p part[p*width + j], fixed order
  for (int j = threadIdx.x; j < width; j += blockDim.x) {
    double s = 0;
    for (int p = 0; p < nparts; ++p) s += part[(int64_t)p * width + j];
    out[j] = s;
  }
}

static int ew_grid(int64_t total, int threads) {
  int64_t g = (total + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

}  // namespace sf

using namespace sf;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* sf_last_error(void) { return g_err.c_str(); }
int32_t sf_version(void) { return 1; }

int64_t sf_group_norm_workspace(int32_t frames, int32_t n_inner, int32_t C) {
  return (int64_t)frames * gn_splits(frames, n_inner) * C * (int64_t)sizeof(double2);
}

sf_status sf_group_norm_stats(sf_view_t x, int32_t frames, int32_t n_inner, int32_t C, int32_t groups, float eps,
                              void* work, float* mean, float* rstd, void* stream) {
  SF_CHECK_ARG(frames >= 1 && n_inner >= 1 && C >= 8 && C % 8 == 0, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(groups >= 1 && C % groups == 0, SF_ERR_PARAM, "groups must divide channels");
  SF_CHECK_ARG(view_vec8_ok(x) && work && mean && rstd, SF_ERR_PARAM, "unaligned view or null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  static const bool direct_on = !(getenv("SF_GN_DIRECT") && getenv("SF_GN_DIRECT")[0] == '0');   // A/B knob
  if (const int gpb = direct_on ? gn_direct_gpb(C, groups, n_inner) : 0) {
    const int W = gpb * (C / groups), nv = W / 8, rpi = 256 / nv;
    const size_t smem = (size_t)rpi * W * sizeof(double2);
    static size_t set = 48 * 1024;
    if (smem > set) {
      cudaFuncSetAttribute(gn_stats_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      set = smem;
    }
    launch_k(gn_stats_direct_kernel, dim3((unsigned)(groups / gpb), (unsigned)frames), dim3(rpi * nv), smem, st, x,
             n_inner, C, groups, gpb, eps, mean, rstd);
    return launch_status("sf_group_norm_stats");
  }
  int splits = gn_splits(frames, n_inner);
  int nvec = C / 8;
  int threads = nvec <= 256 ? (256 / nvec) * nvec : 256;
  size_t smem = nvec <= 256 ? (size_t)(256 / nvec) * C * sizeof(double2) : 0;
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(gn_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  launch_k(gn_partial_kernel, dim3(frames * splits), dim3(threads), smem, st, x, n_inner, C, splits, (double2*)work);
  launch_gn_finalize((const double2*)work, frames, splits, C, groups, (int64_t)n_inner * (C / groups), eps, mean,
                     rstd, st);
  return launch_status("sf_group_norm_stats");
}

int32_t sf_conv_gn_splits(int32_t H, int32_t W) {
  if (H < 1 || W < 1) return 0;
  return conv_tiling(H, W).gn_splits();
}

sf_status sf_conv_gn_partials(sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C, void* partial,
                              void* stream) {
  SF_CHECK_ARG(frames >= 1 && H >= 1 && W >= 1 && C >= 2 && C % 2 == 0, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(y.ptr && partial && (y.ld % 2) == 0 && ((uintptr_t)y.ptr & 3) == 0 && ((uintptr_t)partial & 7) == 0,
               SF_ERR_PARAM, "null or unaligned buffer");
  return conv_gn_partials(y, frames, H, W, C, partial, (cudaStream_t)stream);
}

sf_status sf_group_norm_finalize(const void* partial, int32_t frames, int32_t splits, int32_t n_inner, int32_t C,
                                 int32_t groups, float eps, float* mean, float* rstd, void* stream) {
  SF_CHECK_ARG(frames >= 1 && splits >= 1 && n_inner >= 1 && C >= 1, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(groups >= 1 && C % groups == 0, SF_ERR_PARAM, "groups must divide channels");
  SF_CHECK_ARG(partial && mean && rstd && ((uintptr_t)partial & 7) == 0, SF_ERR_PARAM, "null or unaligned buffer");
  launch_gn_finalize((const float2*)partial, frames, splits, C, groups, (int64_t)n_inner * (C / groups), eps, mean,
                     rstd, (cudaStream_t)stream);
  return launch_status("sf_group_norm_finalize");
}

sf_status sf_group_norm_apply(sf_view_t x, sf_view_t y, int32_t frames, int32_t n_inner, int32_t C, int32_t groups,
                              const float* mean, const float* rstd, const float* gamma, const float* beta,
                              int32_t act, void* stream) {
  SF_CHECK_ARG(frames >= 1 && n_inner >= 1 && C % 8 == 0, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(groups >= 1 && C % groups == 0, SF_ERR_PARAM, "groups must divide channels");
  SF_CHECK_ARG(view_vec8_ok(x) && view_vec8_ok(y), SF_ERR_PARAM, "unaligned view");
  SF_CHECK_ARG(aligned16(gamma) && aligned16(beta), SF_ERR_PARAM, "gamma/beta must be 16-byte aligned");
  const int nvec = C / 8;
  const int threads = nvec <= 256 ? (256 / nvec) * nvec : 256;
  static int occ = 0;
  if (!occ) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gn_apply_kernel, 256, 0);
    if (occ < 1) occ = 1;
  }
  // persistent: every resident block gets an equal share (>= ~32 rows per thread)
  const int64_t rows = (int64_t)frames * n_inner;
  const int rpi = nvec <= 256 ? 256 / nvec : 1;
  int64_t grid = (int64_t)num_sms() * occ;
  const int64_t most = (rows + rpi * 8 - 1) / (rpi * 8);
  if (grid > most) grid = most;
  if (grid < 1) grid = 1;
  launch_k(gn_apply_kernel, dim3((unsigned)grid), dim3(threads), 0, (cudaStream_t)stream, x, y, frames, n_inner, C, groups, mean, rstd,
                                                                        gamma, beta, act);
  return launch_status("sf_group_norm_apply");
}

static sf_status layer_norm_launch(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C,
                                   const float* gamma, const float* beta, float eps, int32_t act, float2* stats,
                                   void* stream);

sf_status sf_layer_norm(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C, const float* gamma,
                        const float* beta, float eps, int32_t act, void* stream) {
  SF_CHECK_ARG(view_vec8_ok(y), SF_ERR_PARAM, "unaligned view");
  SF_CHECK_ARG(aligned16(gamma) && aligned16(beta), SF_ERR_PARAM, "gamma/beta must be 16-byte aligned");
  return layer_norm_launch(x, y, n_outer, n_inner, C, gamma, beta, eps, act, nullptr, stream);
}

sf_status sf_layer_norm_stats(sf_view_t x, int32_t n_outer, int32_t n_inner, int32_t C, float eps, float* stats,
                              void* stream) {
  SF_CHECK_ARG(stats && ((uintptr_t)stats & 7) == 0, SF_ERR_PARAM, "stats must be 8-byte aligned");
  return layer_norm_launch(x, sf_view_t{nullptr, 8, 0}, n_outer, n_inner, C, nullptr, nullptr, eps, 0,
                           reinterpret_cast<float2*>(stats), stream);
}

static sf_status layer_norm_launch(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C,
                                   const float* gamma, const float* beta, float eps, int32_t act, float2* stats,
                                   void* stream) {
  SF_CHECK_ARG(n_outer >= 1 && n_inner >= 1 && C % 8 == 0 && C <= 32 * 8 * 12, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(view_vec8_ok(x), SF_ERR_PARAM, "unaligned view");
  const int64_t rows = (int64_t)n_outer * n_inner;
  cudaStream_t st = (cudaStream_t)stream;
  const int nvec = C / 8;
  // lanes per row: enough that every lane holds <= vmax vectors (<= 12 for the widest rows)
  int L = 1;
  // vectors per lane: 10 (more bytes in flight per warp) measured faster on B200 for 320- and
  // >= 1280-channel rows, 5 for 640 (L2: 22.8 -> 16.7 us, L0: 82 -> 80 us; L1: 41 vs 46 us)
  const int vmax = (nvec >= 160 || nvec <= 40) ? 10 : 5;
  while (L < 32 && (nvec + L - 1) / L > vmax) L *= 2;
  const int vpl = (nvec + L - 1) / L;
  const int64_t warps = (rows + 32 / L - 1) / (32 / L);
  const int64_t g = (warps * 32 + 255) / 256;
  // persistent grid (3-4 resident blocks per SM, see __launch_bounds__): every block walks rows
  // with a stride of the whole grid.  Packed rows: L0 (320 ch) 74 -> 59 us, L1 41.5 -> 37 us; a
  // register prefetch of the next row group (128 registers, 2 blocks per SM) measured slower
  const int64_t cap = (int64_t)num_sms() * (vpl <= 5 ? 4 : 3);
  const int grid = (int)(g < cap ? (g < 1 ? 1 : g) : cap);
  const size_t smem = stats ? 16 : (size_t)C * 2 * sizeof(float);
#define SF_LN(LL, VV) \
  launch_k(layer_norm_kernel<LL, VV>, dim3(grid), dim3(256), smem, st, x, y, n_outer, n_inner, C, gamma, beta, eps, act, \
           stats)
  // the template's VPL must cover vpl = ceil(nvec / L)
  if (L == 1 && vpl > 5) SF_LN(1, 10);
  else if (L == 1) SF_LN(1, 5);
  else if (L == 2 && vpl > 5) SF_LN(2, 10);
  else if (L == 2) SF_LN(2, 5);
  else if (L == 4 && vpl > 5) SF_LN(4, 10);
  else if (L == 4) SF_LN(4, 5);
  else if (L == 8 && vpl > 5) SF_LN(8, 10);
  else if (L == 16 && vpl > 5) SF_LN(16, 10);
  else if (L == 8) SF_LN(8, 5);
  else if (L == 16) SF_LN(16, 5);
  else if (vpl <= 5) SF_LN(32, 5);
  else if (vpl <= 8) SF_LN(32, 8);
  else SF_LN(32, 12);
#undef SF_LN
  return launch_status("sf_layer_norm");
}

sf_status sf_silu(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C, void* stream) {
  SF_CHECK_ARG(n_outer >= 1 && n_inner >= 1 && C % 8 == 0, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(view_vec8_ok(x) && view_vec8_ok(y), SF_ERR_PARAM, "unaligned view");
  int64_t total = (int64_t)n_outer * n_inner * (C / 8);
  launch_k(rows_ew_kernel<EW_SILU>, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, x, y, n_outer, n_inner, C, 0);
  return launch_status("sf_silu");
}

sf_status sf_add(sf_view_t a, sf_view_t b, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C,
                 int32_t b_broadcast_inner, void* stream) {
  SF_CHECK_ARG(n_outer >= 1 && n_inner >= 1 && C % 8 == 0, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(view_vec8_ok(a) && view_vec8_ok(b) && view_vec8_ok(y), SF_ERR_PARAM, "unaligned view");
  int64_t total = (int64_t)n_outer * n_inner * (C / 8);
  launch_k(rows_ew_kernel<EW_ADD>, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, a, b, y, n_outer, n_inner, C,
                                                                                 b_broadcast_inner);
  return launch_status("sf_add");
}

sf_status sf_copy_rows(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C, void* stream) {
  SF_CHECK_ARG(n_outer >= 1 && n_inner >= 1 && C >= 1, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(x.ptr && y.ptr, SF_ERR_PARAM, "null view");
  if (C % 8 || !view_vec8_ok(x) || !view_vec8_ok(y)) {  // odd channel ranges: element copy
    int64_t total = (int64_t)n_outer * n_inner * C;
    launch_k(copy_rows_scalar_kernel, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, y, n_outer, n_inner, C);
    return launch_status("sf_copy_rows");
  }
  int64_t total = (int64_t)n_outer * n_inner * (C / 8);
  launch_k(rows_ew_kernel<EW_COPY>, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, x, y, n_outer, n_inner, C, 0);
  return launch_status("sf_copy_rows");
}

sf_status sf_downsample2x(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C, void* stream) {
  SF_CHECK_ARG(H % 2 == 0 && W % 2 == 0, SF_ERR_SHAPE, "downsample2x needs even h, w");
  SF_CHECK_ARG(frames >= 1 && C % 8 == 0 && view_vec8_ok(x) && view_vec8_ok(y), SF_ERR_PARAM, "bad view");
  int64_t total = (int64_t)frames * (H / 2) * (W / 2) * (C / 8);
  launch_k(downsample_kernel, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, y, frames, H, W, C);
  return launch_status("sf_downsample2x");
}

sf_status sf_upsample2x(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C, void* stream) {
  SF_CHECK_ARG(frames >= 1 && C % 8 == 0 && view_vec8_ok(x) && view_vec8_ok(y), SF_ERR_PARAM, "bad view");
  int64_t total = (int64_t)frames * H * W * (C / 8);   // one thread per input vector
  SF_CHECK_ARG(total < (1ll << 31), SF_ERR_SHAPE, "upsample input too large for 32-bit indexing");
  launch_k(upsample_kernel, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, y, frames, H, W, C);
  return launch_status("sf_upsample2x");
}

sf_status sf_group_norm_project(sf_view_t x, int32_t frames, int32_t n_inner, int32_t C, int32_t groups,
                                const float* mean, const float* rstd, const float* gamma, const float* beta,
                                int32_t act, const void* w, int32_t N, float* out, int64_t ldo, void* stream) {
  SF_CHECK_ARG(frames >= 1 && n_inner >= 16 && C >= 64 && C % 64 == 0 && C <= 384, SF_ERR_SHAPE,
               "C must be a multiple of 64 in [64, 384] (shared memory), frames of >= 16 rows");
  SF_CHECK_ARG(groups >= 1 && C % groups == 0, SF_ERR_PARAM, "groups must divide channels");
  SF_CHECK_ARG(N >= 2 && N <= GP_NP && N % 2 == 0 && ldo >= N && ldo % 2 == 0, SF_ERR_SHAPE,
               "N must be even, <= 48, and fit the output rows");
  SF_CHECK_ARG(view_vec8_ok(x) && aligned16(w) && ((uintptr_t)out & 7) == 0 && mean && rstd && gamma && beta,
               SF_ERR_PARAM, "unaligned or null operand");
  return gn_project_launch(x, frames, n_inner, C, groups, mean, rstd, gamma, beta, act, w, N, out, ldo,
                           (cudaStream_t)stream);
}

sf_status sf_downsample2x_gn(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C,
                             int32_t splits, void* out_part, int32_t out_ld, void* in_part, int32_t in_ld,
                             void* stream) {
  SF_CHECK_ARG(H % 2 == 0 && W % 2 == 0, SF_ERR_SHAPE, "downsample2x needs even h, w");
  SF_CHECK_ARG(frames >= 1 && C % 8 == 0 && view_vec8_ok(x) && view_vec8_ok(y), SF_ERR_PARAM, "bad view");
  SF_CHECK_ARG(splits >= 1 && splits <= (H / 2) * (W / 2), SF_ERR_PARAM, "1 <= splits <= output pixels");
  SF_CHECK_ARG((!out_part || out_ld >= C) && (!in_part || in_ld >= C), SF_ERR_PARAM, "partial row too short");
  return launch_resample_gn(0, x, y, frames, H, W, C, splits, out_part, out_ld, 0, in_part, in_ld,
                            (cudaStream_t)stream);
}

sf_status sf_upsample2x_gn(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C, int32_t splits,
                           void* out_part, int32_t out_ld, int32_t out_c0, void* stream) {
  SF_CHECK_ARG(frames >= 1 && C % 8 == 0 && view_vec8_ok(x) && view_vec8_ok(y), SF_ERR_PARAM, "bad view");
  SF_CHECK_ARG(splits >= 1 && splits <= H * W, SF_ERR_PARAM, "1 <= splits <= input pixels");
  SF_CHECK_ARG(out_part && out_c0 >= 0 && out_ld >= out_c0 + C, SF_ERR_PARAM, "partial row too short");
  return launch_resample_gn(1, x, y, frames, H, W, C, splits, out_part, out_ld, out_c0, nullptr, 0,
                            (cudaStream_t)stream);
}

sf_status sf_softmax_rows(const float* s, int64_t lds, void* p, int64_t ldp, int64_t rows, int32_t n, void* stream) {
  SF_CHECK_ARG(rows >= 1 && n >= 4 && n % 4 == 0 && n <= 256 * 4 * 16, SF_ERR_SHAPE,
               "row length must be a multiple of 4 in [4, 16384]");
  SF_CHECK_ARG(aligned16(s) && lds % 4 == 0 && ldp % 4 == 0, SF_ERR_PARAM, "rows must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int per = (n / 4 + 255) / 256;
  bf16* P = (bf16*)p;
#define SF_SM(K) launch_k(softmax_rows_kernel<K>, dim3((unsigned)rows), dim3(256), 0, st, s, lds, P, ldp, n)
  if (per <= 1) SF_SM(1);
  else if (per <= 2) SF_SM(2);
  else if (per <= 3) SF_SM(3);
  else if (per <= 4) SF_SM(4);
  else if (per <= 9) SF_SM(9);
  else SF_SM(16);
#undef SF_SM
  return launch_status("sf_softmax_rows");
}

bool temporal_core_tc_supported(int T, int C, int koff, int voff, sf_view_t qkv, sf_view_t out);
sf_status temporal_core_tc_launch(sf_view_t qkv, int koff, int voff, sf_view_t out, int B, int T, int n_inner, int C,
                                  float scale, cudaStream_t st);

sf_status sf_temporal_attention_core(sf_view_t qkv, int32_t koff, int32_t voff, sf_view_t out, int32_t B, int32_t T,
                                     int32_t n_inner, int32_t C, float scale, void* stream) {
  SF_CHECK_ARG(B >= 1 && n_inner >= 1 && C >= 1, SF_ERR_SHAPE, "bad extents");
  // 32 < T <= 128: tcgen05 tiles of floor(128 / T) pixels (csrc/temporal_attn_tc.cu)
  if (temporal_core_tc_supported(T, C, koff, voff, qkv, out))
    return temporal_core_tc_launch(qkv, koff, voff, out, B, T, n_inner, C, scale, (cudaStream_t)stream);
  SF_CHECK_ARG(T >= 1 && T <= TA_MAXT, SF_ERR_SHAPE, "temporal attention supports 1 <= T <= 64 (128 on tcgen05)");
  if (T <= 32 && C % 8 == 0 && koff % 8 == 0 && voff % 8 == 0 && view_vec8_ok(qkv) && out.ld % 2 == 0) {
    const int smem = TQ_WARPS * 3 * 32 * TQ_LD * 2;
    static bool init = false;
    if (!init) {
      cudaFuncSetAttribute(temporal_attn_mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(temporal_attn_mma_kernel<TQ_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      init = true;
    }
    const int64_t pixels = (int64_t)B * n_inner;
    const float sl2 = scale * 1.4426950408889634f;
    // fewer pixels than ~8 warps per SM (C3 L2 / L3: 576 / 144): one block per pixel, channels split
    if (pixels < (int64_t)num_sms() * 8 && C >= 2 * TQ_CH)
      launch_k(temporal_attn_mma_kernel<TQ_WARPS>, dim3((unsigned)pixels), dim3(TQ_WARPS * 32), smem,
               (cudaStream_t)stream, qkv, koff, voff, out, B, T, n_inner, C, sl2);
    else
      launch_k(temporal_attn_mma_kernel<1>, dim3((unsigned)((pixels + TQ_WARPS - 1) / TQ_WARPS)),
               dim3(TQ_WARPS * 32), smem, (cudaStream_t)stream, qkv, koff, voff, out, B, T, n_inner, C, sl2);
    return launch_status("sf_temporal_attention_core");
  }
  launch_k(temporal_attn_kernel, dim3(B * n_inner), dim3(256), 0, (cudaStream_t)stream, qkv, koff, voff, out, T, n_inner, C, scale);
  return launch_status("sf_temporal_attention_core");
}

sf_status sf_conv3x3_smallcin(const float* x, int32_t frames, int32_t H, int32_t W, int32_t cin, const float* w,
                              const float* bias, int32_t cout, sf_view_t y, void* stream) {
  SF_CHECK_ARG(cin >= 1 && cin <= 16 && cout % 8 == 0 && cout <= 1280, SF_ERR_SHAPE,
               "need cin <= 16, cout % 8 == 0, cout <= 1280");
  SF_CHECK_ARG(view_vec8_ok(y) && aligned16(w) && (cin != 4 || aligned16(x)), SF_ERR_PARAM,
               "unaligned view, weights or latent");
  const size_t smem = (size_t)9 * cin * cout * sizeof(float);
  SF_CHECK_ARG(smem <= 200 * 1024, SF_ERR_SHAPE, "in_conv weights exceed shared memory");
  cudaStream_t st = (cudaStream_t)stream;
  // tensor-core path: K = 9*cin padded to 16, whole cout resident in smem
  if (cout % SCM_NCH == 0 && cout <= 640 && 9 * cin <= 96) {
    const int kp = (9 * cin + 15) / 16 * 16;
    if (kp <= 16) return conv_smallcin_mma_launch<16>(x, frames, H, W, cin, w, bias, cout, y, 0, nullptr, st);
    if (kp <= 48) return conv_smallcin_mma_launch<48>(x, frames, H, W, cin, w, bias, cout, y, 0, nullptr, st);
    return conv_smallcin_mma_launch<96>(x, frames, H, W, cin, w, bias, cout, y, 0, nullptr, st);
  }
  if (cout % 32 == 0) {
    static size_t cfg32 = 0;
    if (smem > 48 * 1024 && smem > cfg32) {
      cudaFuncSetAttribute(conv_smallcin_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cfg32 = smem;
    }
    const int64_t total = (int64_t)frames * H * W * (cout / 32);
    launch_k(conv_smallcin_kernel<32>, dim3(ew_grid(total, SC_THREADS)), dim3(SC_THREADS), smem, st, x, frames, H, W, cin, w, bias,
                                                                                   cout, y);
  } else {
    static size_t cfg8 = 0;
    if (smem > 48 * 1024 && smem > cfg8) {
      cudaFuncSetAttribute(conv_smallcin_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cfg8 = smem;
    }
    const int64_t total = (int64_t)frames * H * W * (cout / 8);
    launch_k(conv_smallcin_kernel<8>, dim3(ew_grid(total, SC_THREADS)), dim3(SC_THREADS), smem, st, x, frames, H, W, cin, w, bias,
                                                                                  cout, y);
  }
  return launch_status("sf_conv3x3_smallcin");
}

sf_status sf_conv3x3_smallcin_gn(const float* x, int32_t frames, int32_t H, int32_t W, int32_t cin, const float* w,
                                 const float* bias, int32_t cout, sf_view_t y, int32_t splits, void* part,
                                 void* stream) {
  SF_CHECK_ARG(frames >= 1 && H >= 1 && W >= 1 && cin >= 1, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(cout % SCM_NCH == 0 && cout <= 640 && 9 * cin <= 96, SF_ERR_UNSUPPORTED,
               "GroupNorm partials need the tensor-core in_conv (cout % 64 == 0, <= 640; 9 cin <= 96)");
  SF_CHECK_ARG(splits >= 1 && splits <= (H * W + 15) / 16, SF_ERR_PARAM, "1 <= splits <= 16-pixel tiles per frame");
  SF_CHECK_ARG(x && w && bias && part && view_vec8_ok(y) && ((uintptr_t)part & 7) == 0, SF_ERR_PARAM,
               "null or unaligned operand");
  const int kp = (9 * cin + 15) / 16 * 16;
  cudaStream_t st = (cudaStream_t)stream;
  if (kp <= 16) return conv_smallcin_mma_launch<16>(x, frames, H, W, cin, w, bias, cout, y, splits, part, st);
  if (kp <= 48) return conv_smallcin_mma_launch<48>(x, frames, H, W, cin, w, bias, cout, y, splits, part, st);
  return conv_smallcin_mma_launch<96>(x, frames, H, W, cin, w, bias, cout, y, splits, part, st);
}

sf_status sf_conv3x3_tapsum(const float* y, int32_t ldy, int32_t frames, int32_t H, int32_t W, int32_t cout,
                            const float* bias, sf_view_t out, void* stream) {
  SF_CHECK_ARG(frames >= 1 && H >= 1 && W >= 1 && cout >= 1 && ldy >= 9 * cout, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(y && out.ptr, SF_ERR_PARAM, "null buffer");
  const int64_t total = (int64_t)frames * H * W * cout;
  launch_k(conv_tapsum_kernel, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, y, ldy, frames, H, W, cout, bias, out);
  return launch_status("sf_conv3x3_tapsum");
}

sf_status sf_gemv_f32(const float* W, const float* e, const float* b, float* y, int32_t N, int32_t K, void* stream) {
  SF_CHECK_ARG(N >= 1 && K >= 1, SF_ERR_SHAPE, "bad extents");
  launch_k(gemv_kernel, dim3((N * 32 + 255) / 256), dim3(256), 0, (cudaStream_t)stream, W, e, b, y, N, K);
  return launch_status("sf_gemv_f32");
}

sf_status sf_bcthw_to_rows_f32(const float* x, float* y, int32_t frames, int32_t C, int32_t HW, void* stream) {
  int64_t total = (int64_t)frames * C * HW;
  launch_k(transpose_f32_kernel, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, y, frames, C, HW, 1);
  return launch_status("sf_bcthw_to_rows_f32");
}

sf_status sf_rows_to_bcthw_f32(const float* x, float* y, int32_t frames, int32_t C, int32_t HW, void* stream) {
  int64_t total = (int64_t)frames * C * HW;
  launch_k(transpose_f32_kernel, dim3(ew_grid(total, 256)), dim3(256), 0, (cudaStream_t)stream, x, y, frames, HW, C, 0);
  return launch_status("sf_rows_to_bcthw_f32");
}

sf_status sf_axpy_f32(float* x, const float* eps, float alpha, int64_t n, void* stream) {
  launch_k(axpy_kernel, dim3(ew_grid(n, 256)), dim3(256), 0, (cudaStream_t)stream, x, eps, alpha, n);
  return launch_status("sf_axpy_f32");
}

int64_t sf_dot3_workspace(int64_t n) { return (int64_t)DOT_BLOCKS * 3 * sizeof(double); }

sf_status sf_dot3_bf16(const void* a, const void* b, int64_t n, void* work, double* out, void* stream) {
  SF_CHECK_ARG(n >= 1 && aligned16(a) && aligned16(b), SF_ERR_PARAM, "bad probe buffers");
  cudaStream_t st = (cudaStream_t)stream;
  launch_k(dot3_partial_kernel, dim3(DOT_BLOCKS), dim3(DOT_THREADS), 0, st, (const bf16*)a, (const bf16*)b, n, (double*)work);
  launch_k(sum_parts_kernel, dim3(1), dim3(32), 0, st, (const double*)work, DOT_BLOCKS, 3, out);
  return launch_status("sf_dot3_bf16");
}


}  // extern "C"
