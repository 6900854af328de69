// sf_gemm: host-side validation (mirrors kernels.py:327-328: validate before
// compute) and backend selection between the tcgen05/TMA kernel and the
// mma.sync fallback.
#include "common.cuh"

namespace sf {
sf_status gemm_mma_launch(const sf_gemm_args& p, cudaStream_t st);
bool gemm_tc_supported(const sf_gemm_args& p);
sf_status gemm_tc_launch(const sf_gemm_args& p, cudaStream_t st);
sf_status conv_gn_partials(sf_view_t y, int frames, int H, int W, int N, void* part, cudaStream_t st);
}  // namespace sf

using namespace sf;

static sf_status validate(const sf_gemm_args* a) {
  SF_CHECK_ARG(a != nullptr, SF_ERR_PARAM, "null args");
  SF_CHECK_ARG(a->mode >= SF_GEMM_PLAIN && a->mode <= SF_GEMM_TCONV3, SF_ERR_PARAM, "unknown mode");
  SF_CHECK_ARG(a->n_outer >= 1 && a->n_inner >= 1 && a->N >= 1 && a->cin >= 1 && a->batch >= 1, SF_ERR_SHAPE,
               "empty extents");
  SF_CHECK_ARG(a->cin % 8 == 0, SF_ERR_SHAPE, "cin must be a multiple of 8");
  SF_CHECK_ARG(a->a.ptr && a->w && a->out.ptr, SF_ERR_PARAM, "null operand");
  SF_CHECK_ARG(view_vec8_ok(a->a), SF_ERR_PARAM, "A view must be 16-byte aligned with ld % 8 == 0");
  SF_CHECK_ARG(aligned16(a->w) && a->w_ld % 8 == 0, SF_ERR_PARAM, "W must be 16-byte aligned with ld % 8 == 0");
  if (!a->w_kmajor) SF_CHECK_ARG(a->N % 8 == 0, SF_ERR_SHAPE, "MN-major W needs N % 8 == 0");
  if (a->mode == SF_GEMM_CONV3X3)
    SF_CHECK_ARG(a->H >= 1 && a->W >= 1 && (int64_t)a->H * a->W == a->n_inner, SF_ERR_SHAPE,
                 "conv3x3: n_inner must equal H*W");
  if (a->mode == SF_GEMM_TCONV3)
    SF_CHECK_ARG(a->T >= 1 && a->n_outer % a->T == 0, SF_ERR_SHAPE, "tconv: n_outer must be a multiple of T");
  SF_CHECK_ARG(a->act == SF_ACT_NONE || a->act == SF_ACT_SILU, SF_ERR_PARAM, "unknown activation");
  if (a->rowstats)
    SF_CHECK_ARG(a->colvec && a->mode == SF_GEMM_PLAIN && a->batch == 1 && ((uintptr_t)a->rowstats & 7) == 0,
                 SF_ERR_PARAM, "folded LayerNorm needs colvec, PLAIN mode, batch 1, 8-byte aligned stats");
  if (a->gn_partial)
    SF_CHECK_ARG(a->mode == SF_GEMM_CONV3X3 && !a->out_fp32 && a->N % 2 == 0 && aligned16(a->gn_partial),
                 SF_ERR_PARAM, "GroupNorm partials need CONV3X3, bf16 output, even N, 16-byte aligned buffer");
  return SF_OK;
}

extern "C" int32_t sf_gemm_backend(const sf_gemm_args* a) {
  if (validate(a) != SF_OK) return 0;
  const int be = a->backend & ~SF_GEMM_NO_PAIR;
  if (be == 1) return 1;
  if (be == 2) return gemm_tc_supported(*a) ? 2 : 0;
  return gemm_tc_supported(*a) ? 2 : 1;
}

extern "C" sf_status sf_gemm(const sf_gemm_args* a, void* stream) {
  sf_status s = validate(a);
  if (s != SF_OK) return s;
  int be = sf_gemm_backend(a);
  SF_CHECK_ARG(be != 0, SF_ERR_UNSUPPORTED, "forced tcgen05 backend cannot take this shape");
  if (be == 2) return gemm_tc_launch(*a, (cudaStream_t)stream);
  s = gemm_mma_launch(*a, (cudaStream_t)stream);
  // the mma.sync kernel has no fused statistics: the same partials from a pass over its output
  if (s == SF_OK && a->gn_partial)
    s = conv_gn_partials(a->out, a->n_outer, a->H, a->W, a->N, a->gn_partial, (cudaStream_t)stream);
  return s;
}
