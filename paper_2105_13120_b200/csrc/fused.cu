// Fused RSA kernels (placeholder until the tcgen05 attention kernels land).
#include "common.h"

extern "C" {
int rsa_fused_supported(const rsa_geom*) { return 0; }
int rsa_fwd_stats(const rsa_geom*, rsa_view, rsa_view, float*, int, void*) {
  return rsa::fail(RSA_ERR_UNSUPPORTED, "fused kernels not built");
}
int rsa_fwd_probs_pv(const rsa_geom*, rsa_view, rsa_view, rsa_view, const float*, int, rsa_view, rsa_view, int,
                     rsa_view, void*) {
  return rsa::fail(RSA_ERR_UNSUPPORTED, "fused kernels not built");
}
int rsa_bwd_dkdv(const rsa_geom*, rsa_view, rsa_view, rsa_view, rsa_view, const float*, rsa_view, rsa_view, rsa_view,
                 int, int, void*) {
  return rsa::fail(RSA_ERR_UNSUPPORTED, "fused kernels not built");
}
int rsa_bwd_dq(const rsa_geom*, rsa_view, rsa_view, rsa_view, int, rsa_view, void*) {
  return rsa::fail(RSA_ERR_UNSUPPORTED, "fused kernels not built");
}
}
