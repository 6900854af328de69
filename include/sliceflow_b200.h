/*
 * sliceflow_b200 -- C ABI of the sm_100a kernels behind the sliced + grouped +
 * rehash denoising path of Streamlined Inference (arXiv 2411.01171).
 *
 * Drop-in boundary.  The reference (`sliceflow`, pure numpy) has no FFI: its
 * hot path sits behind plain Python functions, all of which bottom out in
 * `apply_kernel` (reference kernels.py:323-368).  Every entry point below
 * replaces one reference kernel or one fused chain of them; the mapping is
 * cited per function.  The Python package `paper_2411_01171_b200` binds these
 * through ctypes and mirrors the reference's
 * `apply_kernel` / `execute_group` / `execute` / `rehash_execute` /
 * `run_denoise` signatures on top.
 *
 * Conventions
 *   - Plain pointers to DEVICE memory, sizes in elements, a cudaStream_t passed
 *     as void*.  No torch types.  Nothing allocates; callers own all memory.
 *   - Activations are bf16, channels-last: a row is the C contiguous channels
 *     of one (b, t, h, w) position.  Rows are addressed through sf_view_t, a
 *     two-level row view: row (o, i) lives at  ptr + (o*ostride + i)*ld.
 *     A spatial slice (a frame range) is o = frame, i = pixel; a temporal slice
 *     (a pixel band) is o = b*T+t, i = pixel within the band.  Channel ranges
 *     of a wider buffer (zero-copy concat) are just ptr offset + larger ld.
 *   - Statistics/accumulation are fp32 (fp64 for similarity dot products).
 *   - Every function validates shapes/params on the host BEFORE launching
 *     (mirrors kernels.py:327-328) and returns an sf_status:
 *        SF_OK, SF_ERR_SHAPE (-> ShapeMismatch), SF_ERR_PARAM (-> InvalidParam),
 *        SF_ERR_CUDA (-> SliceflowError, exit 1), SF_ERR_UNSUPPORTED.
 *     sf_last_error() returns a message for the most recent failure on the
 *     calling thread.
 *   - All kernels are deterministic (fixed reduction order, no float atomics):
 *     an all-key rehash schedule reproduces the plain run bit for bit
 *     (SPEC.md:428).
 */
#ifndef SLICEFLOW_B200_H
#define SLICEFLOW_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SF_OK = 0,
  SF_ERR_SHAPE = 1,
  SF_ERR_PARAM = 2,
  SF_ERR_CUDA = 3,
  SF_ERR_UNSUPPORTED = 4
} sf_status;

/* Two-level row view: row (o, i) at ptr + (o*ostride + i)*ld elements. */
typedef struct {
  void* ptr;
  int64_t ld;       /* elements between rows of one outer block            */
  int64_t ostride;  /* rows between consecutive outer blocks               */
} sf_view_t;

/* GEMM A-operand addressing modes. */
typedef enum {
  SF_GEMM_PLAIN = 0,   /* A[m][k] = row m                                     */
  SF_GEMM_CONV3X3 = 1, /* implicit im2col, 3x3 taps, zero pad 1 (kernels.py:181-201) */
  SF_GEMM_TCONV3 = 2   /* 3 taps along t, zero pad 1 (kernels.py:204-225)     */
} sf_gemm_mode;

typedef enum { SF_ACT_NONE = 0, SF_ACT_SILU = 1 } sf_act;

#define SF_GEMM_NO_PAIR 4   /* sf_gemm_args.backend flag */

/*
 * Implicit GEMM  out[m][n] = act( sum_k A[m][k] * W[n][k] * alpha + bias[n]
 *                                + rowbias[o(m)][n] ) + res[m][n]
 * M = n_outer * n_inner rows; K = taps * cin (tap-major, channel-minor).
 * CONV3X3: inner = H*W pixels of one frame (o = frame).
 * TCONV3:  o = b*T + t, inner = pixels; tap j reads o + j - 1 within the batch.
 * Batched over `batch` with per-batch element strides *_bstride.
 */
typedef struct {
  int32_t mode;          /* sf_gemm_mode */
  int32_t n_outer, n_inner;
  int32_t H, W, T;       /* conv geometry (CONV3X3: H*W == n_inner; TCONV3: T) */
  int32_t cin;           /* channels per tap */
  int32_t N;             /* output channels  */
  int32_t batch;
  sf_view_t a;           /* bf16 activations */
  int64_t a_bstride;
  const void* w;         /* bf16 [N][taps*cin] K-major, or [K][N] if w_kmajor==0 */
  int32_t w_kmajor;
  int64_t w_ld;          /* row stride of W in elements */
  int64_t w_bstride;
  float alpha;           /* scale on the accumulator (attention 1/sqrt(C)) */
  const float* bias;     /* [N] or NULL */
  const float* rowbias;  /* [n_outer][N] per-frame bias (step embedding) or NULL */
  int64_t rowbias_stride;/* elements between rowbias rows; 0 = broadcast */
  int32_t act;           /* sf_act */
  sf_view_t res;         /* bf16 residual (ptr NULL = none) */
  int64_t res_bstride;
  sf_view_t out;         /* output rows */
  int64_t out_bstride;
  int32_t out_fp32;      /* 1: fp32 output, 0: bf16 */
  int32_t backend;       /* 0 auto, 1 force mma.sync path, 2 force tcgen05 path; | SF_GEMM_NO_PAIR:
                            single-CTA tcgen05 tiles only (no cta_group::2 clusters) */
  /* LayerNorm folded into the GEMM (PLAIN, batch 1): rowstats[2m] = rstd_m, rowstats[2m+1] =
   * -mean_m*rstd_m of A's row m (sf_layer_norm_stats), colvec[n] = sum_k W[n][k]; the accumulator
   * becomes rstd_m * (acc - mean_m * colvec[n]) = LN(A)_m . W_n before alpha / bias / act / res.
   * NULL = off. */
  const float* rowstats;
  const float* colvec;
  /* GroupNorm statistics of the output from the epilogue (CONV3X3, bf16 output): per (frame,
   * split, channel) fp32 (sum, sum of squares) of the STORED bf16 values, layout
   * [n_outer][sf_conv_gn_splits(H, W)][N] float2; a split = one half (64 rows) of a 128-pixel
   * tile, or one frame's rows of a tail tile.  Finished by sf_group_norm_finalize.  NULL = off.
   * Replaces the statistics pass of the GroupNorm that reads this conv's output
   * (kernels.py:228-237; unet.py:191-193, res.conv1 -> res.norm2). */
  void* gn_partial;
} sf_gemm_args;

/* ---- GEMM core: conv2d / temporal_conv / linear / attention projections ---- */
/* replaces kernels.py:181-201 (_conv2d), 204-225 (_temporal_conv),
 * 256-266 (_linear), 285-291 (attention matmuls)                          */
sf_status sf_gemm(const sf_gemm_args* args, void* stream);
/* Which backend sf_gemm would pick (1 = mma.sync, 2 = tcgen05/TMA). */
int32_t sf_gemm_backend(const sf_gemm_args* args);

/* ---- normalisation (kernels.py:228-253) ---- */
/* GroupNorm statistics per (frame, group) over (C/groups channels x n_inner rows):
 * mean and rstd = 1/sqrt(var + eps), biased variance.  work: fp32 scratch of
 * sf_group_norm_workspace() bytes. */
int64_t sf_group_norm_workspace(int32_t frames, int32_t n_inner, int32_t C);
sf_status sf_group_norm_stats(sf_view_t x, int32_t frames, int32_t n_inner, int32_t C, int32_t groups,
                              float eps, void* work, float* mean, float* rstd, void* stream);
/* Partial-sum splits per frame of a CONV3X3 sf_gemm with gn_partial (frame-geometry only). */
int32_t sf_conv_gn_splits(int32_t H, int32_t W);
/* The same partials as a pass over a stored conv output y (frames of H x W rows, C channels):
 * identical layout and summation order (the mma.sync backend's path, and the fused one's checker). */
sf_status sf_conv_gn_partials(sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C, void* partial,
                              void* stream);
/* mean / rstd per (frame, group) from [frames][splits][C] float2 (sum, sum sq) partials,
 * fp64 fixed-order combine; n_inner = rows per frame. */
sf_status sf_group_norm_finalize(const void* partial, int32_t frames, int32_t splits, int32_t n_inner, int32_t C,
                                 int32_t groups, float eps, float* mean, float* rstd, void* stream);
/* out[r][n] = sum_c act(GN(x))[r][c] * w[n][c] (w bf16 [N][C], N even <= 48, fp32 out rows of ldo):
 * the GroupNorm apply (+ SiLU) fused into a narrow projection -- the per-tap projection of the
 * network's out_conv (kernels.py:228-253 then 181-201), so the normalised tensor never reaches HBM. */
sf_status sf_group_norm_project(sf_view_t x, int32_t frames, int32_t n_inner, int32_t C, int32_t groups,
                                const float* mean, const float* rstd, const float* gamma, const float* beta,
                                int32_t act, const void* w, int32_t N, float* out, int64_t ldo, void* stream);
/* y = act((x - mean) * rstd * gamma + beta), per (frame, group) stats. */
sf_status sf_group_norm_apply(sf_view_t x, sf_view_t y, int32_t frames, int32_t n_inner, int32_t C,
                              int32_t groups, const float* mean, const float* rstd, const float* gamma,
                              const float* beta, int32_t act, void* stream);
/* Per-row LayerNorm statistics for a folded GEMM: stats[2r] = rstd, stats[2r+1] = -mean*rstd
 * (two-pass, same arithmetic as sf_layer_norm). */
sf_status sf_layer_norm_stats(sf_view_t x, int32_t n_outer, int32_t n_inner, int32_t C, float eps, float* stats,
                              void* stream);
/* LayerNorm over the C channels of every row (kernels.py:240-244), optional SiLU. */
sf_status sf_layer_norm(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C,
                        const float* gamma, const float* beta, float eps, int32_t act, void* stream);

/* ---- elementwise / boundary (kernels.py:247-253, 311-365) ---- */
sf_status sf_silu(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C, void* stream);
/* y = a + b; b may be a per-outer bias row (b_rows_broadcast=1: row (o,i) reads b row o). */
sf_status sf_add(sf_view_t a, sf_view_t b, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C,
                 int32_t b_broadcast_inner, void* stream);
/* strided channel-range copy (concat operand placement, split) */
sf_status sf_copy_rows(sf_view_t x, sf_view_t y, int32_t n_outer, int32_t n_inner, int32_t C, void* stream);
/* 2x2 mean pool (x00+x01+x10+x11)*0.25, frames of H x W -> H/2 x W/2 */
sf_status sf_downsample2x(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C,
                          void* stream);
/* nearest-neighbour x2, frames of H x W -> 2H x 2W */
sf_status sf_upsample2x(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C,
                        void* stream);
/* The same resampling, also writing GroupNorm partials (float2 (sum, sum sq) per (frame, split,
 * channel) at part[(frame * splits + split) * ld + c0 + c]; split = a contiguous range of the
 * coarse pixels) for the GroupNorm that reads the result, or (downsample, in_part) the skip tensor
 * it reads (unet.py:221-244: downsample -> next res.norm1; skip and upsample halves of
 * up_blocks.i.concat -> res.norm1).  Finished by sf_group_norm_finalize.  NULL part = off. */
sf_status sf_downsample2x_gn(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C,
                             int32_t splits, void* out_part, int32_t out_ld, void* in_part, int32_t in_ld,
                             void* stream);
sf_status sf_upsample2x_gn(sf_view_t x, sf_view_t y, int32_t frames, int32_t H, int32_t W, int32_t C, int32_t splits,
                           void* out_part, int32_t out_ld, int32_t out_c0, void* stream);

/* ---- attention cores (kernels.py:269-308) ---- */
/* Row softmax of fp32 scores S[rows][n] (already scaled) -> bf16 P[rows][n]. */
sf_status sf_softmax_rows(const float* s, int64_t lds, void* p, int64_t ldp, int64_t rows, int32_t n,
                          void* stream);
/* Fused spatial attention core (flash, tcgen05/TMEM): per frame,
 * out = softmax(q k^T * scale) v over HW tokens, head_dim C in {128,192,256,320}.
 * q, k: bf16 row views (o = frame, i = token) sharing one row stride; vt: bf16
 * V^T [frames][C][HW]. */
int32_t sf_flash_supported(int32_t HW, int32_t C);
sf_status sf_spatial_attention_core(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int32_t frames,
                                    int32_t HW, int32_t C, float scale, void* stream);
/* Temporal attention core per pixel: q|k|v rows (o = b*T+t, i = pixel), q at
 * column 0, k at qkv_koff, v at qkv_voff of view qkv; writes softmax(q k^T *
 * scale) v into out.  T <= 32: mma.sync; 32 < T <= 128 with C, koff, voff
 * multiples of 64: tcgen05; otherwise SIMT (T <= 64). */
sf_status sf_temporal_attention_core(sf_view_t qkv, int32_t koff, int32_t voff, sf_view_t out, int32_t B,
                                     int32_t T, int32_t n_inner, int32_t C, float scale, void* stream);
/* Whole temporal attention op, fused (tcgen05/TMEM; replaces the QKV projection, the core and
 * the output projection of kernels.py:276-308 for one LayerNorm'd input x):
 *   out = softmax(x Mqk x^T) x Mvo  (+ res),  per pixel over its T frames,
 * with w = [Mqk^T ; Mvo^T] bf16 [2C][C] row-major, Mqk = Wq Wk^T log2(e)/sqrt(C), Mvo = Wv Wo.
 * x, res, out: bf16 row views (o = b*T + t, i = pixel).  res may be null.
 * Supported: T <= 128, C in {64, 128, 192, 256, 320}. */
int32_t sf_temporal_attention_fused_supported(int32_t T, int32_t C);
sf_status sf_temporal_attention_fused(sf_view_t x, const void* w, sf_view_t res, sf_view_t out, int32_t B,
                                      int32_t T, int32_t n_inner, int32_t C, void* stream);

/* ---- network edges ---- */
/* in_conv with tiny cin: x fp32 channels-last [frames][H*W][cin] -> bf16 rows */
sf_status sf_conv3x3_smallcin(const float* x, int32_t frames, int32_t H, int32_t W, int32_t cin,
                              const float* w /*[3][3][ci][co] fp32*/, const float* bias, int32_t cout,
                              sf_view_t y, void* stream);
/* out_conv with tiny cout, second half: y holds the per-tap projections
 * Y[f][p][tap*cout + co] = x[f][p] . W_tap[co] (fp32, row stride ldy, written by
 * sf_gemm with the tap-major weight matrix); this sums the 9 shifted taps with
 * zero padding: out[f][p][co] = bias[co] + sum_tap Y[f][p + off(tap)][tap*cout + co]
 * (kernels.py:181-201 regrouped; fixed tap order).  out: fp32 rows view. */
/* in_conv with the GroupNorm partials of its output (the statistics of down_blocks.0.res.norm1,
 * unet.py:213-216): part[(frame * splits + split) * cout + c] = (sum, sum sq) of the stored bf16 values
 * over the split's contiguous run of 16-pixel tiles.  Tensor-core path only (cout % 64 == 0). */
sf_status sf_conv3x3_smallcin_gn(const float* x, int32_t frames, int32_t H, int32_t W, int32_t cin, const float* w,
                                 const float* bias, int32_t cout, sf_view_t y, int32_t splits, void* part,
                                 void* stream);
sf_status sf_conv3x3_tapsum(const float* y, int32_t ldy, int32_t frames, int32_t H, int32_t W, int32_t cout,
                            const float* bias, sf_view_t out, void* stream);
/* y[n] = W[n][:] . e + b[n] for a batch of step embeddings (res-block emb_proj) */
sf_status sf_gemv_f32(const float* W, const float* e, const float* b, float* y, int32_t N, int32_t K,
                      void* stream);
/* (b,t,c,h,w) fp32 <-> channels-last fp32 */
sf_status sf_bcthw_to_rows_f32(const float* x, float* y, int32_t frames, int32_t C, int32_t HW, void* stream);
sf_status sf_rows_to_bcthw_f32(const float* x, float* y, int32_t frames, int32_t C, int32_t HW, void* stream);
/* latent update x <- x - alpha * eps */
sf_status sf_axpy_f32(float* x, const float* eps, float alpha, int64_t n, void* stream);

/* ---- Step Rehash (kernels.py:375-390) ---- */
/* out[0..2] = (a.a, b.b, a.b) over n bf16 elements, fp64 accumulation in a
 * fixed order.  work: sf_dot3_workspace(n) bytes. */
int64_t sf_dot3_workspace(int64_t n);
sf_status sf_dot3_bf16(const void* a, const void* b, int64_t n, void* work, double* out, void* stream);
/* Gram matrix of K probes (pointers in a device array), fp64 out[K][K]. */
int64_t sf_gram_workspace(int32_t K, int64_t n);
sf_status sf_gram_bf16(const void* const* probes, int32_t K, int64_t n, void* work, double* out, void* stream);

/* ---- misc ---- */
const char* sf_last_error(void);
int32_t sf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SLICEFLOW_B200_H */
