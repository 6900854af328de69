// C ABI of the fused spatial attention core (kernels.py:269-300).
// Kernels: flash_attn5.cu (CTA pairs, 96/128-key blocks, P over S in TMEM: the
// default) and flash_attn2.cu (single CTA; head dim 192 and single-query-tile frames).
#include "common.cuh"

#include <cstdlib>
#include <mutex>

namespace sf {
sf_status flash2_launch(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int frames, int HW, int C,
                        float scale, cudaStream_t st);
sf_status flash5_launch(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int frames, int HW, int C,
                        float scale, cudaStream_t st);
bool flash5_supported(int C);

static bool encode_available() {
  static int ok = -1;
  if (ok < 0) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    ok = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
         q == cudaDriverEntryPointSuccess;
  }
  return ok == 1;
}
}  // namespace sf

using namespace sf;

extern "C" int32_t sf_flash_supported(int32_t HW, int32_t C) {
  return (C == 320 || C == 256 || C == 192 || C == 128) && HW >= 64 && encode_available();
}

extern "C" sf_status sf_spatial_attention_core(sf_view_t q, sf_view_t k, const void* vt, sf_view_t out, int32_t frames,
                                               int32_t HW, int32_t C, float scale, void* stream) {
  SF_CHECK_ARG(frames >= 1 && HW >= 1, SF_ERR_SHAPE, "bad extents");
  SF_CHECK_ARG(sf_flash_supported(HW, C), SF_ERR_UNSUPPORTED, "fused attention needs C in {128,192,256,320}");
  SF_CHECK_ARG(view_vec8_ok(q) && view_vec8_ok(k) && view_vec8_ok(out) && aligned16(vt) && HW % 8 == 0,
               SF_ERR_PARAM, "operands must be 16-byte aligned, HW % 8 == 0");
  SF_CHECK_ARG(q.ld == k.ld, SF_ERR_PARAM, "q and k must share a row stride");
  cudaStream_t st = (cudaStream_t)stream;
  // SF_FLASH=2 forces the single-CTA kernel (A/B runs); default: v5 CTA pairs where possible
  static const char* ver = getenv("SF_FLASH");
  const int v = ver ? atoi(ver) : 5;
  if (v >= 5 && flash5_supported(C) && (HW + 127) / 128 >= 2) return flash5_launch(q, k, vt, out, frames, HW, C, scale, st);
  return flash2_launch(q, k, vt, out, frames, HW, C, scale, st);
}
