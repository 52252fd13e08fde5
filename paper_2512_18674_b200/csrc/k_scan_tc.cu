// k_scan_tc.cu -- S2+S3 on the 5th-generation tensor cores (tcgen05).  (stub: filled next)
#include "tc_host.h"

namespace remoe {

remoe_status_t tc_plan_create(TcPlan* t, const uint16_t* x, int64_t n_rows, int dim, int num_sms,
                              int max_k) {
  (void)x; (void)n_rows; (void)dim; (void)num_sms; (void)max_k;
  t->ok = false;
  t->why = "tensor-core scan not built yet";
  t->grid = 0;
  t->threads_per_cta_queries = 0;
  return REMOE_OK;
}

void tc_plan_destroy(TcPlan* t) { t->ok = false; }

remoe_status_t tc_scan(TcPlan*, const uint16_t*, const float*, int, int, float, const float*, int64_t,
                       int64_t, uint64_t*, uint64_t*, cudaStream_t, int*) {
  return REMOE_ERR_UNSUPPORTED;
}

}  // namespace remoe
