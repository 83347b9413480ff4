// kvp_tc.cu — tensor-core (tcgen05) cross term for large d.  (stub: filled in next)
#include "common.cuh"

namespace falkon {

bool tc_supported(const falkon_ctx *ctx, int kernel, int64_t d) { return false; }

int tc_prepare(falkon_ctx *ctx, const float *X, int64_t n, int64_t d, const float *C, int64_t m,
               double sigma, const double *mu, Prepared *pp) {
  return fail(FALKON_EUNSUPPORTED, "tensor path not built");
}
int tc_pass(falkon_ctx *ctx, const Prepared &pp, bool passA, const float *z, double *out64,
            float *out32) {
  return fail(FALKON_EUNSUPPORTED, "tensor path not built");
}

}  // namespace falkon
