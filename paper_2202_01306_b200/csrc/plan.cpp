// plan.cpp -- swap plan, ledger and event-driven estimate (see plan.hpp).
//
// Parity target: the non-compute items of simulator._build_items must equal
// ours row for row (key, tensor, channel, resources, nbytes, gpu), and
// hm_plan_simulate must reproduce simulator._run's start/end times exactly.
#include "plan.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <queue>
#include <tuple>

namespace hm {

namespace {

const char *kTensorName[8] = {"X", "Y", "dX", "dY", "W", "dW", "K", "sX"};

// ceil(nbytes * 1e9 / bw) without overflow (simulator.py:45-46 uses bigints).
int64_t xfer_ns(int64_t nbytes, int64_t bw) {
  __int128 num = (__int128)nbytes * 1000000000 + (bw - 1);
  return (int64_t)(num / bw);
}

struct Ctx {
  const hm_machine *m;
  const hm_profile *p;
  int32_t N;
  int64_t pcie, swap_bw, p2p_bw;

  int64_t table(const int64_t *t, int32_t layer, int32_t u, const char *what) const {
    if (layer < 0 || layer >= p->layers)
      throw Error{HM_ERR_MISSING_PROFILE, std::string("no ") + what + " model for layer " + std::to_string(layer)};
    if (u < 0 || u > p->u_top)
      throw Error{HM_ERR_PROFILE_RANGE, std::string(what) + ": microbatch " + std::to_string(u) + " outside table"};
    int64_t v = t[(int64_t)layer * (p->u_top + 1) + u];
    if (v == -1)
      throw Error{HM_ERR_MISSING_PROFILE, std::string("no ") + what + " model for layer " + std::to_string(layer)};
    if (v == -2)
      throw Error{HM_ERR_PROFILE_RANGE, "microbatch " + std::to_string(u) + " above fitted maximum for " + what};
    return v;
  }
  int64_t scalar(const int64_t *t, int32_t layer, const char *what) const {
    if (layer < 0 || layer >= p->layers || t[layer] < 0)
      throw Error{HM_ERR_MISSING_PROFILE, std::string("no ") + what + " for layer " + std::to_string(layer)};
    return t[layer];
  }
  // simulator.py:118-130
  int64_t entry_bytes(int32_t tensor, int32_t layer, const hm_entry &e, int32_t u) const {
    switch (tensor) {
      case HM_W: return scalar(p->w, layer, "weight size");
      case HM_DW: return scalar(p->dw, layer, "gradient size");
      case HM_K: return scalar(p->k, layer, "optimizer-state size");
      default: break;
    }
    if (e.src_layer >= 0) return table(p->y, e.src_layer, u, "output-size");
    if (tensor == HM_X || tensor == HM_SX || tensor == HM_DX) return table(p->x, layer, u, "input-size");
    return table(p->y, layer, u, "output-size");
  }
  int64_t pack_time(const int64_t *t, int32_t lo, int32_t hi, int32_t u, const char *what) const {
    if (!t) throw Error{HM_ERR_MISSING_PROFILE, "profile has no time tables"};
    int64_t s = 0;
    for (int32_t L = lo; L <= hi; ++L) s += table(t, L, u, what);
    return s;
  }
  // simulator.py:133-147
  // sharded Harmony-DP update: (shard params, pack params) of a U task, or {-1, -1}
  std::pair<int64_t, int64_t> update_shard(const TaskInfo &t) const {
    if (!m->dp_sharded_update || t.type != HM_TASK_U) return {-1, -1};
    int64_t P = 0;
    for (int32_t L = t.lo; L <= t.hi; ++L) {
      const int64_t w = scalar(p->w, L, "weight size"), k = scalar(p->k, L, "optimizer-state size");
      if (w % 4 || k != 2 * w)
        throw Error{HM_ERR_VALIDATION, "sharded update needs fp32 weights and K = 2 W (Adam m, v) for layer " +
                                           std::to_string(L)};
      P += w / 4;
    }
    int64_t off, len;
    dp_shard(P, N, t.dev_id, &off, &len);
    return {len, P};
  }
  int64_t compute_ns(const TaskInfo &t, int32_t u) const {
    if (t.type == HM_TASK_F) return pack_time(p->t_f, t.lo, t.hi, u, "time F");
    if (t.type == HM_TASK_B) {
      int64_t d = pack_time(p->t_b, t.lo, t.hi, u, "time B");
      if (t.recompute) d += pack_time(p->t_f, t.lo, t.hi, u, "time F");
      return d;
    }
    int64_t d = 0;
    if (m->cpu_offload_update) {
      for (int32_t L = t.lo; L <= t.hi; ++L) d += xfer_ns(scalar(p->w, L, "weight size"), m->update_cpu_rate);
    } else {
      for (int32_t L = t.lo; L <= t.hi; ++L) d += table(p->t_u, L, 1, "time U");
    }
    const auto sh = update_shard(t);
    if (sh.second > 0) d = d * sh.first / sh.second;  // the shard's share of the pack
    return d;
  }
  int32_t res(int32_t kind, int32_t gpu) const { return kind * N + gpu; }
};

struct Builder {
  Plan &plan;
  Ctx &c;
  int32_t seq = 0;

  int32_t add(int32_t task, int32_t stage, int32_t member, std::initializer_list<int32_t> res,
              int64_t duration, bool compute, int32_t tensor, int32_t channel, int64_t nbytes,
              int32_t gpu) {
    Item it;
    hm_item &r = it.rec;
    r.task = task; r.stage = stage; r.member = member; r.seq = ++seq;
    r.is_compute = compute ? 1 : 0;
    r.tensor = tensor; r.channel = channel; r.gpu = gpu;
    r.layer = -1; r.peer_task = -1; r.peer_member = -1;
    r.n_res = 0;
    for (int32_t x : res) r.res[r.n_res++] = x;
    r.nbytes = nbytes; r.duration_ns = duration; r.start_ns = -1; r.end_ns = -1;
    plan.items.push_back(std::move(it));
    return (int32_t)plan.items.size() - 1;
  }
  void link(int32_t dep, int32_t item, bool at_start = false) {
    if (dep < 0) return;
    plan.items[dep].dependents.push_back({item, at_start});
    plan.items[item].pending += 1;
    plan.items[item].deps.push_back({dep, at_start});
  }
  void p2p_res(int32_t src, int32_t dst, int32_t out[4], int32_t &n) const {
    n = 0;
    out[n++] = c.res(HM_RES_P2P_OUT, src);
    out[n++] = c.res(HM_RES_P2P_IN, dst);
    if (c.m->p2p_group_of[src] != c.m->p2p_group_of[dst]) {
      out[n++] = c.res(HM_RES_ROOT_IN, 0);
      out[n++] = c.res(HM_RES_ROOT_OUT, 0);
    }
  }
  int32_t add_p2p(int32_t task, int32_t member, int32_t src_gpu, int32_t gpu, int64_t nbytes,
                  int32_t tensor) {
    int32_t r[4], n;
    p2p_res(src_gpu, gpu, r, n);
    int64_t bw = (n == 2) ? c.p2p_bw : c.swap_bw;
    int32_t id = add(task, 0, member, {}, xfer_ns(nbytes, bw), false, tensor, HM_PEER2PEER, nbytes, gpu);
    hm_item &rec = plan.items[id].rec;
    rec.n_res = n;
    for (int i = 0; i < n; ++i) rec.res[i] = r[i];
    return id;
  }

  void build() {
    std::vector<int32_t> first_compute(plan.tasks.size(), -1);
    plan.member_computes.assign(plan.tasks.size(), {});
    // mp_out keyed by (src task, dst task, layer) -> legs, insertion order
    std::map<std::tuple<int32_t, int32_t, int32_t>, std::vector<int32_t>> mp_out;
    std::map<std::pair<int32_t, int32_t>, int32_t> prev_on_device;  // (kind, id) -> task

    for (const TaskInfo &t : plan.tasks) {
      const int32_t gpu = t.dev_id;
      auto pit = prev_on_device.find({t.dev_kind, t.dev_id});
      const int32_t prev = pit == prev_on_device.end() ? -1 : pit->second;
      const bool is_update = t.type == HM_TASK_U;

      std::vector<int32_t> task_inputs, gate_first;
      std::map<int32_t, std::vector<int32_t>> member_gate;
      std::vector<std::pair<int32_t, bool>> shm_deps;
      std::vector<std::pair<int32_t, int64_t>> swap_bytes;  // tensor -> bytes, insertion order

      // ---- inputs, grouped by tensor in insertion order -------------------
      size_t i = 0;
      while (i < t.inputs.size()) {
        const int32_t tensor = t.inputs[i].tensor;
        std::vector<std::pair<int32_t, int64_t>> p2p_by_src;                 // src -> bytes
        std::vector<std::pair<int32_t, std::vector<int64_t>>> p2p_aligned;  // src -> per member
        std::vector<int32_t> p2p_layer;  // first layer seen per aligned src (addressing)
        std::vector<int32_t> p2p_by_src_layer;
        for (; i < t.inputs.size() && t.inputs[i].tensor == tensor; ++i) {
          const hm_entry &e = t.inputs[i];
          if (e.channel == HM_CPU_GPU_SWAP) {
            // bf16 swap-payload mode: a forward task moves the bf16 high halves
            // plus the fp32-read prefix of each layer (hm_profile.w_f)
            int64_t b = (tensor == HM_W && t.type == HM_TASK_F && c.p->w_f)
                            ? c.scalar(c.p->w_f, e.layer, "forward weight size")
                            : c.entry_bytes(tensor, e.layer, e, t.group[0]);
            auto f = std::find_if(swap_bytes.begin(), swap_bytes.end(),
                                  [&](auto &kv) { return kv.first == tensor; });
            if (f == swap_bytes.end()) swap_bytes.push_back({tensor, b});
            else f->second += b;
          } else if (e.channel == HM_SHARED_MEMORY) {
            const TaskInfo &src = plan.tasks.at(e.peer_task);
            shm_deps.push_back({e.peer_task, src.group == t.group});
          } else if (e.channel == HM_MESSAGE_PASSING) {
            int64_t nbytes = 0;
            for (int32_t u : t.group) nbytes += c.entry_bytes(tensor, e.layer, e, u);
            if (nbytes == 0) {
              gate_first.push_back(plan.member_computes.at(e.peer_task).back());
              continue;
            }
            int32_t it = add(t.index, 0, 0, {c.res(HM_RES_SWAP_IN, gpu), c.res(HM_RES_ROOT_OUT, 0)},
                             xfer_ns(nbytes, c.swap_bw), false, tensor, HM_MESSAGE_PASSING, nbytes, gpu);
            plan.items[it].rec.layer = e.layer;
            plan.items[it].rec.peer_task = e.peer_task;
            auto legs = mp_out.find({e.peer_task, t.index, e.layer});
            if (legs != mp_out.end())
              for (int32_t leg : legs->second) link(leg, it);
            task_inputs.push_back(it);
          } else if (e.channel == HM_PEER2PEER) {
            const TaskInfo &src = plan.tasks.at(e.peer_task);
            if (src.group == t.group) {
              auto f = std::find_if(p2p_aligned.begin(), p2p_aligned.end(),
                                    [&](auto &kv) { return kv.first == e.peer_task; });
              if (f == p2p_aligned.end()) {
                p2p_aligned.push_back({e.peer_task, std::vector<int64_t>(t.group.size(), 0)});
                p2p_layer.push_back(e.layer);
                f = p2p_aligned.end() - 1;
              }
              for (size_t g = 0; g < t.group.size(); ++g) f->second[g] += c.entry_bytes(tensor, e.layer, e, t.group[g]);
            } else {
              int64_t s = 0;
              for (int32_t u : t.group) s += c.entry_bytes(tensor, e.layer, e, u);
              auto f = std::find_if(p2p_by_src.begin(), p2p_by_src.end(),
                                    [&](auto &kv) { return kv.first == e.peer_task; });
              if (f == p2p_by_src.end()) { p2p_by_src.push_back({e.peer_task, s}); p2p_by_src_layer.push_back(e.layer); }
              else f->second += s;
            }
          } else {
            throw Error{HM_ERR_VALIDATION, "unknown channel kind"};
          }
        }
        for (size_t a = 0; a < p2p_aligned.size(); ++a) {
          const int32_t src = p2p_aligned[a].first;
          const int32_t src_gpu = plan.tasks[src].dev_id;
          for (size_t g = 0; g < p2p_aligned[a].second.size(); ++g) {
            const int64_t nbytes = p2p_aligned[a].second[g];
            if (nbytes == 0) {
              member_gate[(int32_t)g].push_back(plan.member_computes.at(src)[g]);
              continue;
            }
            int32_t it = add_p2p(t.index, (int32_t)g, src_gpu, gpu, nbytes, tensor);
            plan.items[it].rec.layer = p2p_layer[a];
            plan.items[it].rec.peer_task = src;
            plan.items[it].rec.peer_member = (int32_t)g;
            link(plan.member_computes.at(src)[g], it);
            member_gate[(int32_t)g].push_back(it);
          }
        }
        for (size_t a = 0; a < p2p_by_src.size(); ++a) {
          const int32_t src = p2p_by_src[a].first;
          const int64_t nbytes = p2p_by_src[a].second;
          if (nbytes == 0) {
            gate_first.push_back(plan.member_computes.at(src).back());
            continue;
          }
          int32_t it = add_p2p(t.index, 0, plan.tasks[src].dev_id, gpu, nbytes, tensor);
          plan.items[it].rec.layer = p2p_by_src_layer[a];
          plan.items[it].rec.peer_task = src;
          plan.items[it].rec.peer_member = -1;  // whole task
          link(plan.member_computes.at(src).back(), it);
          task_inputs.push_back(it);
        }
      }
      const auto shard = c.update_shard(t);  // sharded DP update: this GPU's K shard only
      if (shard.second >= 0)
        for (auto &kv : swap_bytes)
          if (kv.first == HM_K) kv.second = 8 * shard.first;
      // task-level swap-ins sorted by tensor name (simulator.py:251-260)
      std::stable_sort(swap_bytes.begin(), swap_bytes.end(), [](auto &a, auto &b) {
        return std::strcmp(kTensorName[a.first], kTensorName[b.first]) < 0;
      });
      for (auto &kv : swap_bytes) {
        if (kv.second == 0) continue;
        task_inputs.push_back(add(t.index, 0, 0, {c.res(HM_RES_SWAP_IN, gpu), c.res(HM_RES_ROOT_OUT, 0)},
                                  xfer_ns(kv.second, c.swap_bw), false, kv.first, HM_CPU_GPU_SWAP,
                                  kv.second, gpu));
      }
      // prefetch window (simulator.py:262-269)
      int32_t window = -1;
      if (is_update) {
        if (t.index >= 1) window = first_compute[t.index - 1];
      } else if (prev >= 0) {
        window = first_compute[prev];
      }
      for (int32_t it : task_inputs) link(window, it, true);

      // ---- member computes (simulator.py:271-302) -------------------------
      std::vector<int32_t> computes;
      const int32_t rk = t.dev_kind == HM_DEV_CPU ? HM_RES_UPDATE : HM_RES_COMPUTE;
      std::vector<int32_t> members = is_update ? std::vector<int32_t>{1} : t.group;
      for (size_t g = 0; g < members.size(); ++g) {
        int32_t it = add(t.index, 1, (int32_t)g, {c.res(rk, gpu)}, c.compute_ns(t, members[g]), true,
                         -1, -1, 0, gpu);
        if (g == 0) {
          if (prev >= 0) link(plan.member_computes[prev].back(), it);
          for (int32_t d : task_inputs) link(d, it);
          for (int32_t d : gate_first) link(d, it);
          for (auto &sd : shm_deps)
            if (!sd.second) link(plan.member_computes.at(sd.first).back(), it);
        } else {
          link(computes[g - 1], it);
        }
        for (auto &sd : shm_deps)
          if (sd.second) link(plan.member_computes.at(sd.first).at(g), it);
        auto mg = member_gate.find((int32_t)g);
        if (mg != member_gate.end())
          for (int32_t d : mg->second) link(d, it);
        computes.push_back(it);
      }
      plan.member_computes[t.index] = computes;
      first_compute[t.index] = computes[0];
      prev_on_device[{t.dev_kind, t.dev_id}] = t.index;

      // ---- outputs (simulator.py:304-335) ---------------------------------
      std::vector<std::pair<int32_t, int64_t>> swap_out;
      for (const hm_entry &e : t.outputs) {
        if (e.channel == HM_MESSAGE_PASSING) {
          for (size_t g = 0; g < t.group.size(); ++g) {
            int64_t nbytes = c.entry_bytes(e.tensor, e.layer, e, t.group[g]);
            if (nbytes == 0) continue;
            int32_t it = add(t.index, 2, (int32_t)g, {c.res(HM_RES_SWAP_OUT, gpu), c.res(HM_RES_ROOT_IN, 0)},
                             xfer_ns(nbytes, c.swap_bw), false, e.tensor, HM_MESSAGE_PASSING, nbytes, gpu);
            plan.items[it].rec.layer = e.layer;
            plan.items[it].rec.peer_task = e.peer_task;
            link(computes.at(g), it);
            mp_out[{t.index, e.peer_task, e.layer}].push_back(it);
          }
        } else if (e.channel == HM_CPU_GPU_SWAP) {
          int64_t b = c.entry_bytes(e.tensor, e.layer, e, t.group[0]);
          auto f = std::find_if(swap_out.begin(), swap_out.end(), [&](auto &kv) { return kv.first == e.tensor; });
          if (f == swap_out.end()) swap_out.push_back({e.tensor, b});
          else f->second += b;
        }
      }
      if (shard.second >= 0)
        for (auto &kv : swap_out) {
          if (kv.first == HM_K) kv.second = 8 * shard.first;
          if (kv.first == HM_W) kv.second = 4 * shard.first;
        }
      std::stable_sort(swap_out.begin(), swap_out.end(), [](auto &a, auto &b) {
        return std::strcmp(kTensorName[a.first], kTensorName[b.first]) < 0;
      });
      for (auto &kv : swap_out) {
        if (kv.second == 0) continue;
        int32_t it = add(t.index, 2, 0, {c.res(HM_RES_SWAP_OUT, gpu), c.res(HM_RES_ROOT_IN, 0)},
                         xfer_ns(kv.second, c.swap_bw), false, kv.first, HM_CPU_GPU_SWAP, kv.second, gpu);
        link(computes.back(), it);
      }
    }
  }
};

}  // namespace

Plan *build_plan(const hm_task *tasks, int32_t n_tasks, const int32_t *groups,
                 const hm_entry *entries, const hm_machine *machine, const hm_profile *profile) {
  if (!tasks || n_tasks < 0 || !machine || !profile || !machine->p2p_group_of)
    throw Error{HM_ERR_VALIDATION, "null argument to hm_plan_build"};
  if (machine->pcie_bandwidth <= 0 || machine->root_link_bandwidth <= 0)
    throw Error{HM_ERR_VALIDATION, "bandwidths must be positive"};
  Plan *plan = new Plan();
  plan->gpu_count = machine->gpu_count;
  plan->dp_sharded = machine->dp_sharded_update != 0;
  try {
    plan->tasks.resize(n_tasks);
    for (int32_t i = 0; i < n_tasks; ++i) {
      const hm_task &src = tasks[i];
      TaskInfo &t = plan->tasks[i];
      t.index = src.index; t.type = src.type; t.lo = src.lo; t.hi = src.hi;
      t.dev_kind = src.dev_kind; t.dev_id = src.dev_id; t.recompute = src.recompute;
      if (t.index != i) throw Error{HM_ERR_VALIDATION, "task " + std::to_string(i) + " carries index " + std::to_string(t.index)};
      if (t.dev_id < 0 || t.dev_id >= machine->gpu_count)
        throw Error{HM_ERR_VALIDATION, "task " + std::to_string(i) + " bound to unknown device"};
      if (src.group_len < 1) throw Error{HM_ERR_VALIDATION, "task has an empty group"};
      t.group.assign(groups + src.group_off, groups + src.group_off + src.group_len);
      t.inputs.assign(entries + src.in_off, entries + src.in_off + src.in_len);
      t.outputs.assign(entries + src.out_off, entries + src.out_off + src.out_len);
      for (auto &e : t.inputs)
        if (e.peer_task >= i && e.channel != HM_CPU_GPU_SWAP)
          throw Error{HM_ERR_VALIDATION, "task " + std::to_string(i) + " consumes from a non-earlier task"};
    }
    Ctx c{machine, profile, machine->gpu_count, machine->pcie_bandwidth,
          std::min(machine->pcie_bandwidth, machine->root_link_bandwidth),
          machine->p2p_bandwidth > 0 ? machine->p2p_bandwidth : machine->pcie_bandwidth};
    Builder b{*plan, c};
    b.build();
  } catch (...) {
    delete plan;
    throw;
  }
  return plan;
}

// simulator.py:347-375 -- heap keyed by (ready, key); resources FIFO.
void run_plan(Plan &plan) {
  const int32_t n = (int32_t)plan.items.size();
  const int32_t n_res = 8 * plan.gpu_count;
  std::vector<int64_t> busy(n_res, 0);
  for (auto &it : plan.items) { it.ready = 0; it.pending = 0; it.rec.start_ns = it.rec.end_ns = -1; }
  for (auto &it : plan.items)
    for (auto &e : it.dependents) plan.items[e.child].pending += 1;
  using K = std::tuple<int64_t, int32_t, int32_t, int32_t, int32_t, int32_t>;
  std::priority_queue<K, std::vector<K>, std::greater<K>> heap;
  auto push = [&](int32_t i) {
    const hm_item &r = plan.items[i].rec;
    heap.push(K{plan.items[i].ready, r.task, r.stage, r.member, r.seq, i});
  };
  for (int32_t i = 0; i < n; ++i)
    if (plan.items[i].pending == 0) push(i);
  int32_t done = 0;
  int64_t makespan = 0;
  while (!heap.empty()) {
    K top = heap.top();
    heap.pop();
    Item &it = plan.items[std::get<5>(top)];
    int64_t start = std::get<0>(top);
    for (int r = 0; r < it.rec.n_res; ++r) start = std::max(start, busy[it.rec.res[r]]);
    const int64_t end = start + it.rec.duration_ns;
    for (int r = 0; r < it.rec.n_res; ++r) busy[it.rec.res[r]] = end;
    it.rec.start_ns = start;
    it.rec.end_ns = end;
    makespan = std::max(makespan, end);
    ++done;
    for (const Edge &e : it.dependents) {
      Item &ch = plan.items[e.child];
      ch.ready = std::max(ch.ready, e.at_start ? start : end);
      if (--ch.pending == 0) push(e.child);
    }
  }
  if (done != n)
    throw Error{HM_ERR_DEADLOCK, std::to_string(n - done) +
                                     " work items never became runnable; the task graph has a dependency cycle"};
  plan.makespan = makespan;
  plan.simulated = true;
}

}  // namespace hm
