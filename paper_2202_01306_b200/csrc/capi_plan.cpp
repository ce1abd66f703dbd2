// capi_plan.cpp -- extern "C" entry points of the swap plan (harmony_b200.h).
#include <cstring>
#include <string>

#include "plan.hpp"
#include "runtime/common.hpp"

#include <atomic>

namespace hm {
static thread_local std::string g_last_error;
void set_last_error(const std::string &msg) { g_last_error = msg; }
KernelProfiler *&profiler() {
  static thread_local KernelProfiler *p = nullptr;
  return p;
}
std::atomic<int64_t> &launch_counter() {
  static std::atomic<int64_t> n{0};
  return n;
}
}  // namespace hm

extern "C" {

const char *hm_last_error(void) { return hm::g_last_error.c_str(); }

int64_t hm_launch_count(void) { return hm::launch_counter().load(); }

const char *hm_version(void) { return "harmony_b200 0.1 (sm_100a)"; }

hm_plan *hm_plan_build(const hm_task *tasks, int32_t n_tasks, const int32_t *groups,
                       const hm_entry *entries, const hm_machine *machine,
                       const hm_profile *profile, int32_t *status) {
  try {
    hm::Plan *p = hm::build_plan(tasks, n_tasks, groups, entries, machine, profile);
    if (status) *status = HM_OK;
    return new hm_plan{p};
  } catch (const hm::Error &e) {
    hm::set_last_error(e.msg);
    if (status) *status = e.code;
  } catch (const std::exception &e) {
    hm::set_last_error(std::string("internal: ") + e.what());
    if (status) *status = HM_ERR_INTERNAL;
  }
  return nullptr;
}

int hm_plan_simulate(hm_plan *plan, int64_t *makespan_ns) {
  if (!plan) { hm::set_last_error("null plan"); return HM_ERR_VALIDATION; }
  try {
    hm::run_plan(*plan->p);
    if (makespan_ns) *makespan_ns = plan->p->makespan;
    return HM_OK;
  } catch (const hm::Error &e) {
    hm::set_last_error(e.msg);
    return e.code;
  }
}

int32_t hm_plan_item_count(const hm_plan *plan) { return plan ? (int32_t)plan->p->items.size() : 0; }

int hm_plan_items(const hm_plan *plan, hm_item *out, int32_t cap) {
  if (!plan || !out) { hm::set_last_error("null argument"); return HM_ERR_VALIDATION; }
  const auto &items = plan->p->items;
  if (cap < (int32_t)items.size()) { hm::set_last_error("buffer too small"); return HM_ERR_VALIDATION; }
  for (size_t i = 0; i < items.size(); ++i) out[i] = items[i].rec;
  return (int)items.size();
}

int32_t hm_plan_edge_count(const hm_plan *plan) {
  if (!plan) return 0;
  int32_t n = 0;
  for (auto &it : plan->p->items) n += (int32_t)it.deps.size();
  return n;
}

int hm_plan_edges(const hm_plan *plan, int32_t *dep, int32_t *item, int32_t *at_start, int32_t cap) {
  if (!plan) { hm::set_last_error("null plan"); return HM_ERR_VALIDATION; }
  int32_t n = 0;
  const auto &items = plan->p->items;
  for (size_t i = 0; i < items.size(); ++i)
    for (auto &d : items[i].deps) {
      if (n >= cap) { hm::set_last_error("buffer too small"); return HM_ERR_VALIDATION; }
      dep[n] = d.first; item[n] = (int32_t)i; at_start[n] = d.second ? 1 : 0;
      ++n;
    }
  return n;
}

void hm_plan_free(hm_plan *plan) {
  if (!plan) return;
  delete plan->p;
  delete plan;
}

}  // extern "C"
