// hg_exec.cpp -- graph executor (placeholder until the planner lands)
#include "../../include/hegpu.h"
#include "hg_internal.hpp"

namespace hg {
void set_last_error(const std::string& s);
}

extern "C" {
static int nyi() {
  hg::set_last_error("graph execution not implemented yet");
  return HG_E_INTERNAL;
}
int hg_plan_create(hg_context*, const hg_keys*, const char*, int64_t, uint64_t, hg_plan**) { return nyi(); }
void hg_plan_destroy(hg_plan*) {}
int hg_plan_bind_input(hg_plan*, const char*, const double*, int64_t) { return nyi(); }
int hg_plan_run(hg_plan*) { return nyi(); }
int hg_plan_output(hg_plan*, const char*, double*, int64_t, int64_t*) { return nyi(); }
int hg_plan_output_info(hg_plan*, const char*, int64_t*, int*, double*) { return nyi(); }
int hg_plan_output_ciphertexts(hg_plan*, const char*, uint64_t*, int) { return nyi(); }
int hg_plan_input_info(hg_plan*, const char*, int64_t*, int*) { return nyi(); }
int hg_plan_set_input_ciphertexts(hg_plan*, const char*, const uint64_t*, int) { return nyi(); }
int hg_plan_profile_json(hg_plan*, char*, size_t) { return nyi(); }
int64_t hg_plan_launches(const hg_plan*) { return 0; }
}
