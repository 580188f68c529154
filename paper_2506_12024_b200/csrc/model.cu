// Device decoder (placeholder until the decode step lands).
#include "fq_internal.cuh"
using namespace fqc;
extern "C" {
#define FQ_TODO return guarded([&] { fail(FQ_E_STATE, "fq_model: not implemented yet"); })
fq_status fq_model_create(fq_ctx*, const fq_model_config*, fq_model**) { FQ_TODO; }
fq_status fq_model_destroy(fq_model*) { FQ_TODO; }
fq_status fq_model_num_linears(const fq_model*, int32_t*) { FQ_TODO; }
fq_status fq_model_linear_id(const fq_model*, int32_t, char*, int32_t) { FQ_TODO; }
fq_status fq_model_linear_index(const fq_model*, const char*, int32_t*) { FQ_TODO; }
fq_status fq_model_linear(fq_model*, int32_t, fq_layer**) { FQ_TODO; }
fq_status fq_model_set_param(fq_model*, const char*, const float*, int64_t) { FQ_TODO; }
fq_status fq_model_init_random(fq_model*, uint64_t, float) { FQ_TODO; }
fq_status fq_model_set_rung(fq_model*, int32_t, int32_t, int32_t) { FQ_TODO; }
fq_status fq_model_get_rung(const fq_model*, int32_t, int32_t, int32_t*) { FQ_TODO; }
fq_status fq_model_set_all_rungs(fq_model*, int32_t, int32_t) { FQ_TODO; }
fq_status fq_model_reset_slot(fq_model*, int32_t) { FQ_TODO; }
fq_status fq_model_slot_length(const fq_model*, int32_t, int64_t*) { FQ_TODO; }
fq_status fq_model_prefill(fq_model*, int32_t, const int32_t*, int64_t, float*, fq_row_stats*) { FQ_TODO; }
fq_status fq_model_decode(fq_model*, int32_t, const int32_t*, const int32_t*, float*, fq_row_stats*) { FQ_TODO; }
fq_status fq_model_logits(fq_model*, float**) { FQ_TODO; }
fq_status fq_model_step_bytes(const fq_model*, int32_t, const int32_t*, int64_t*, int64_t*) { FQ_TODO; }
fq_status fq_model_calibrate_logit_kl(fq_model*, const int32_t*, int64_t, int64_t, int32_t, int32_t, double*, double*) { FQ_TODO; }
}
