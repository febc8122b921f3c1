// Temporary: entry points whose kernels land in later commits.
#include "trg_internal.cuh"
using namespace trg;
extern "C" {
int trg_build_tree(trg_ctx*, const double*, size_t, int, const trg_model_config*, trg_tree_dev**,
                   trg_build_diag*) {
  set_error("trg_build_tree: not built yet");
  return TRG_ERUNTIME;
}
int trg_register_clouds(trg_ctx*, const double*, size_t, const double*, size_t, int,
                        const trg_reg_config*, trg_reg_result*) {
  set_error("trg_register_clouds: not built yet");
  return TRG_ERUNTIME;
}
}
