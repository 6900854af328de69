// GroupNorm (+ SiLU) in ONE cooperative kernel (kernels.py:228-237, 247-253).
//
// The split version (gn_partial -> gn_finalize -> gn_apply) costs three launches per
// GroupNorm and, at the deeper levels, is dominated by launch gaps and tails: a C3 key step
// spends 1.4 ms in 60 GroupNorm launches for 4.3 GB of traffic (0.66 ms at HBM peak).  Here a
// persistent grid of exactly the resident blocks runs the three phases back to back,
// separated by two grid barriers (co-residency guaranteed by the cooperative launch):
//   A  per (frame, row split): fp32 partial sums of x and x^2 per channel -> fp64 partials;
//   B  per (frame, group), one warp: fixed-order fp64 sum of its splits x channels -> mean, rstd;
//   C  y = act(x * (rstd*gamma) + (beta - mean*rstd*gamma)), equal contiguous row shares.
// Phase C re-reads x; at the levels whose activation fits the 126 MB L2 that read is an L2 hit.
// Every reduction has a fixed order: bitwise reproducible.
#include "common.cuh"

namespace sf {
namespace gnf {

constexpr int THREADS = 256, U = 8;

struct Barrier {
  unsigned count, gen;
};

__device__ __forceinline__ void grid_barrier(Barrier* b) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(&b->gen) : "memory");
    __threadfence();
    if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
      b->count = 0;
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&b->gen) : "memory");
    } else {
      unsigned now;
      do {
        __nanosleep(64);
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(now) : "l"(&b->gen) : "memory");
      } while (now == g);
    }
  }
  __syncthreads();
}

struct Args {
  sf_view_t x, y;
  int frames, n_inner, C, groups, splits, act;
  float eps;
  const float* gamma;
  const float* beta;
  double2* partial;   // [frames][splits][C]
  float* mean;        // [frames * groups]
  float* rstd;
  Barrier* bar;
};

__device__ void partial_item(const Args& a, int frame, int split, double2* red) {
  const int C = a.C, nvec = C / 8;
  const bool wide = nvec > THREADS;          // > 2048 channels: one vector per thread, no row groups
  const int rpi = wide ? 1 : THREADS / nvec;
  const int chunk = (a.n_inner + a.splits - 1) / a.splits;
  const int r0 = split * chunk, r1 = min(a.n_inner, r0 + chunk);
  const int lane_r = wide ? 0 : (int)threadIdx.x / nvec;
  const bool active = wide || lane_r < rpi;
  for (int vb = wide ? (int)threadIdx.x : (int)threadIdx.x % nvec; vb < nvec; vb += wide ? THREADS : nvec) {
    float s[8], q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = q[j] = 0.f;
    if (active) {
      int r = r0 + lane_r;
      for (; r + (U - 1) * rpi < r1; r += U * rpi) {
        bf16x8 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[u] = *reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(a.x, frame, r + u * rpi) + vb * 8);
        float fs[8], fq[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) fs[j] = fq[j] = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float f[8];
          unpack8(v[u], f);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            fs[j] += f[j];
            fq[j] = fmaf(f[j], f[j], fq[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[j] += fs[j];
          q[j] += fq[j];
        }
      }
      for (; r < r1; r += rpi) {
        float f[8];
        unpack8(*reinterpret_cast<const bf16x8*>(row_ptr<const bf16>(a.x, frame, r) + vb * 8), f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[j] += f[j];
          q[j] = fmaf(f[j], f[j], q[j]);
        }
      }
    }
    double2* out = a.partial + ((int64_t)frame * a.splits + split) * C + vb * 8;
    if (wide) {
#pragma unroll
      for (int j = 0; j < 8; ++j) out[j] = make_double2((double)s[j], (double)q[j]);
    } else {
      if (active) {
#pragma unroll
        for (int j = 0; j < 8; ++j) red[lane_r * C + vb * 8 + j] = make_double2((double)s[j], (double)q[j]);
      }
    }
  }
  if (!wide) {
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += THREADS) {
      double ss = 0, qq = 0;
      for (int rr = 0; rr < rpi; ++rr) {
        const double2 t = red[rr * C + c];
        ss += t.x;
        qq += t.y;
      }
      a.partial[((int64_t)frame * a.splits + split) * C + c] = make_double2(ss, qq);
    }
    __syncthreads();
  }
}

__device__ void finalize_items(const Args& a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = THREADS / 32;
  const int cg = a.C / a.groups, items = a.frames * a.groups, per = a.splits * cg;
  const double count = (double)a.n_inner * cg;
  for (int it = blockIdx.x * wpb + warp; it < items; it += gridDim.x * wpb) {
    const int f = it / a.groups, g = it % a.groups;
    const double2* base = a.partial + (int64_t)f * a.splits * a.C + g * cg;
    double s = 0, q = 0;
    for (int k = lane; k < per; k += 32) {
      const int sp = k / cg, c = k % cg;
      const double2 t = base[(int64_t)sp * a.C + c];
      s += t.x;
      q += t.y;
    }
    s = warp_sum_d(s);
    q = warp_sum_d(q);
    if (lane == 0) {
      const double mu = s / count;
      double var = q / count - mu * mu;
      if (var < 0) var = 0;
      a.mean[it] = (float)mu;
      a.rstd[it] = (float)(1.0 / sqrt(var + (double)a.eps));
    }
  }
}

__device__ void apply_rows(const Args& a) {
  const int C = a.C, cg = C / a.groups, nvec = C / 8;
  const bool wide = nvec > THREADS;
  const int rpi = wide ? 1 : THREADS / nvec;
  const int64_t total = (int64_t)a.frames * a.n_inner;
  const int64_t r0 = total * blockIdx.x / gridDim.x, r1 = total * (blockIdx.x + 1) / gridDim.x;
  const int lr = wide ? 0 : (int)threadIdx.x / nvec;
  if (lr >= rpi) return;
  for (int v = wide ? (int)threadIdx.x : (int)threadIdx.x % nvec; v < nvec; v += wide ? THREADS : nvec) {
    for (int64_t seg = r0; seg < r1;) {
      const int f = (int)(seg / a.n_inner);
      const int64_t seg_end = min(r1, (int64_t)(f + 1) * a.n_inner);
      const int i0 = (int)(seg - (int64_t)f * a.n_inner), i1 = (int)(seg_end - (int64_t)f * a.n_inner);
      seg = seg_end;
      float ss[8], bb[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = v * 8 + j, g = c / cg;
        ss[j] = a.rstd[f * a.groups + g] * __ldg(a.gamma + c);
        bb[j] = fmaf(-a.mean[f * a.groups + g], ss[j], __ldg(a.beta + c));
      }
      const bf16* src = row_ptr<const bf16>(a.x, f, 0) + v * 8;
      bf16* dst = row_ptr<bf16>(a.y, f, 0) + v * 8;
      const int64_t xld = a.x.ld, yld = a.y.ld;
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
            fv[j] = a.act ? silu_f(t) : t;
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
          fv[j] = a.act ? silu_f(t) : t;
        }
        *reinterpret_cast<bf16x8*>(dst + (int64_t)i * yld) = pack8(fv);
      }
    }
  }
}

__global__ void __launch_bounds__(THREADS, 2) gn_fused_kernel(const __grid_constant__ Args a) {
  griddep_wait();
  griddep_trigger();
  extern __shared__ double2 red[];
  const int items = a.frames * a.splits;
  for (int it = blockIdx.x; it < items; it += gridDim.x) partial_item(a, it / a.splits, it % a.splits, red);
  __threadfence();
  grid_barrier(a.bar);
  finalize_items(a);
  __threadfence();
  grid_barrier(a.bar);
  apply_rows(a);
}

static int smem_bytes(int C) {
  const int nvec = C / 8;
  return nvec > THREADS ? 0 : (THREADS / nvec) * C * (int)sizeof(double2);
}

static int grid_size(int C) {
  // every resident block (two per SM: 256 threads, <= 32 KB of shared memory each)
  static int occ[2] = {0, 0};
  const int big = smem_bytes(C) > 0 ? 1 : 0;
  if (!occ[big]) {
    cudaFuncSetAttribute(gn_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, gn_fused_kernel, THREADS, big ? 32 * 1024 : 0);
    occ[big] = o < 1 ? 1 : (o > 2 ? 2 : o);
  }
  return num_sms() * occ[big];
}

static int splits_for(int frames, int n_inner, int grid) {
  int s = (grid + frames - 1) / frames;     // about one (frame, split) item per block
  const int most = (n_inner + 31) / 32;     // >= 32 rows per split
  if (s > most) s = most;
  return s < 1 ? 1 : s;
}

}  // namespace gnf
}  // namespace sf

using namespace sf;

extern "C" {

int64_t sf_group_norm_fused_workspace(int32_t frames, int32_t n_inner, int32_t C, int32_t groups) {
  const int grid = gnf::grid_size(C);
  const int64_t splits = gnf::splits_for(frames, n_inner, grid);
  return (int64_t)frames * splits * C * (int64_t)sizeof(double2) + 2 * (int64_t)frames * groups * sizeof(float);
}

sf_status sf_group_norm(sf_view_t x, sf_view_t y, int32_t frames, int32_t n_inner, int32_t C, int32_t groups,
                        float eps, const float* gamma, const float* beta, int32_t act, void* work, void* barrier,
                        void* stream) {
  SF_CHECK_ARG(frames >= 1 && n_inner >= 1 && C >= 8 && C % 8 == 0, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(groups >= 1 && C % groups == 0, SF_ERR_PARAM, "groups must divide channels");
  SF_CHECK_ARG(view_vec8_ok(x) && view_vec8_ok(y) && work && barrier, SF_ERR_PARAM, "unaligned view or null buffer");
  SF_CHECK_ARG(aligned16(gamma) && aligned16(beta) && aligned16(work), SF_ERR_PARAM, "unaligned parameters");
  gnf::Args a{};
  a.x = x;
  a.y = y;
  a.frames = frames;
  a.n_inner = n_inner;
  a.C = C;
  a.groups = groups;
  a.act = act;
  a.eps = eps;
  a.gamma = gamma;
  a.beta = beta;
  const int grid = gnf::grid_size(C);
  a.splits = gnf::splits_for(frames, n_inner, grid);
  a.partial = (double2*)work;
  a.mean = (float*)((char*)work + (int64_t)frames * a.splits * C * sizeof(double2));
  a.rstd = a.mean + (int64_t)frames * groups;
  a.bar = (gnf::Barrier*)barrier;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gnf::THREADS);
  cfg.dynamicSmemBytes = gnf::smem_bytes(C);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // every block resident: the grid barriers are safe
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, gnf::gn_fused_kernel, a);
  return launch_status("sf_group_norm");
}

}  // extern "C"
