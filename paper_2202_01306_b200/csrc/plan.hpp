// plan.hpp -- the swap plan: work items, their dependencies and the ledger.
//
// Restates the reference's item construction (simulator.py:150-336) and its
// FIFO event loop (simulator.py:347-375) in C++ so the runtime executes the
// very plan the estimator prices.  Items are built in the reference's order
// (task, then inputs / member computes / outputs), which is a topological
// order of the dependency DAG: the executor enqueues them in that order.
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/harmony_b200.h"

namespace hm {

struct Edge {
  int32_t child;
  bool at_start;
};

struct Item {
  hm_item rec{};              // exported record (key, bytes, times, ...)
  std::vector<Edge> dependents;
  int32_t pending = 0;
  int64_t ready = 0;
  std::vector<std::pair<int32_t, bool>> deps;  // (dep item, at_start), for the runtime
};

struct TaskInfo {
  int32_t index, type, lo, hi, dev_kind, dev_id, recompute;
  std::vector<int32_t> group;
  std::vector<hm_entry> inputs, outputs;
};

// Harmony-DP sharded update (hm_machine.dp_sharded_update): GPU g's shard of
// a pack with `params` parameters, in parameters.  Shards are 64-parameter
// aligned (256-B device / host offsets); trailing ranks may get none.
inline int64_t dp_shard_chunk(int64_t params, int32_t n) { return (params + 64 * (int64_t)n - 1) / (64 * (int64_t)n) * 64; }
inline void dp_shard(int64_t params, int32_t n, int32_t g, int64_t *off, int64_t *len) {
  const int64_t c = dp_shard_chunk(params, n);
  *off = std::min<int64_t>((int64_t)g * c, params);
  *len = std::min<int64_t>(c, params - *off);
}

struct Plan {
  int32_t gpu_count = 1;
  bool dp_sharded = false;  // built with hm_machine.dp_sharded_update
  std::vector<TaskInfo> tasks;
  std::vector<Item> items;
  std::vector<std::vector<int32_t>> member_computes;  // per task
  int64_t makespan = 0;
  bool simulated = false;
};

// Throws hm::Error on failure.
struct Error {
  int code;
  std::string msg;
};

Plan *build_plan(const hm_task *tasks, int32_t n_tasks, const int32_t *groups,
                 const hm_entry *entries, const hm_machine *machine, const hm_profile *profile);
void run_plan(Plan &plan);

void set_last_error(const std::string &msg);

}  // namespace hm

struct hm_plan {
  hm::Plan *p;
};
