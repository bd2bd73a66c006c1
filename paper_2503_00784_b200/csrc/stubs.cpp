// Temporary: draft/engine entry points land in draft.cpp / engine.cpp.
#include "../../include/duodec_b200.h"
extern "C" {
int dd_draft_create(const dd_model_desc*, uint64_t, const dd_plant_desc*, int, const int*, int,
                    dd_draft** out) { if (out) *out = nullptr; return DD_E_STATE; }
void dd_draft_destroy(dd_draft*) {}
int dd_draft_logits(dd_draft*, const int32_t*, int, float*) { return DD_E_STATE; }
int dd_draft_time_token(dd_draft*, int, float*) { return DD_E_STATE; }
int dd_engine_run(dd_ctx*, dd_draft*, const dd_engine_config*, const int32_t*, int,
                  dd_generation_result*) { return DD_E_STATE; }
int dd_calibrate(dd_ctx*, dd_draft*, int, int, int, double*, int*) { return DD_E_STATE; }
}
