// efla.cu — probe-batched factorized Lanczos (EFLA) and the SLQ log-likelihood.
#include "../../include/gsgpc.h"

extern "C" {

gsgpc_status gsgpc_factorized_lanczos_fused(gsgpc_ctx*, gsgpc_kg*, gsgpc_stats*, int, const double*, const double*,
                                            const double*, double, int, double*, double*, int32_t*) {
  return GSGPC_UNSUPPORTED;
}

gsgpc_status gsgpc_log_likelihood_gsgp(gsgpc_ctx*, gsgpc_stats*, gsgpc_kg*, double, const gsgpc_loglik_options*,
                                       gsgpc_loglik_result*) {
  return GSGPC_UNSUPPORTED;
}

}  // extern "C"
