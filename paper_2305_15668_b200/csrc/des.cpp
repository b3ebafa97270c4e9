// Round discrete-event simulation -- engine.run_round (engine.py:53-230)
// with the executor manager (executor_manager.py:81-238), the double-pointer
// and greedy schedulers (scheduler.py:40-124), capped max-min sharing
// (cost_model.py:48-87) and the round metrics (metrics.py:129-167).
//
// Bit-exactness contract: every floating-point expression is evaluated in
// the same order as the reference (compiled with -ffp-contract=off), every
// Python `sum()` over floats is reproduced with CPython 3.12's Neumaier
// compensated summation, and all ties break on (time, kind rank, client id
// byte order) exactly as the reference's heap / sort keys do.
//
// Complexity: pending participants are kept pre-sorted by (budget, id) in a
// doubly linked list, so each scheduler call is O(accepted) instead of the
// reference's O(N log N) re-sort per slot-free.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <deque>
#include <queue>
#include <string>
#include <vector>

#include "../../include/fedhc.h"

namespace fedhc {
int fail(int code, const std::string& msg);
}

namespace {

constexpr double kCapacity = 100.0;  // cost_model.py:18
constexpr double kEpsSched = 1e-9;   // scheduler.py:14
constexpr double kEpsWork = 1e-9;    // engine.py:27
constexpr double kEpsTime = 1e-12;   // engine.py:28

// KIND_RANK (metrics.py:21-28)
enum Rank { kLaunched = 0, kPhase = 1, kTrained = 2, kUploaded = 3, kSlotFreed = 4 };
enum TimerKind { kStart = 0, kUploadDone = 3, kSlotFree = 4 };  // value == rank
enum Life { kIdle, kLaunching, kRunning, kTerminating };
enum Instr { kInLaunch = 0, kInStart = 1, kInUpload = 2, kInTerminate = 3 };

// CPython >= 3.12 sum() over a sequence of floats (Neumaier).
struct PySum {
  double s = 0.0, c = 0.0;
  bool any = false;
  void add(double x) {
    any = true;
    const double t = s + x;
    if (fabs(s) >= fabs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
  }
  double value() const {
    double r = s;
    if (c != 0.0 && isfinite(c)) r += c;
    return r;  // empty -> 0 (int 0 in Python; compares identically)
  }
};

double work_units(const fedhc_des_client& w, double alpha, double beta) {
  const double batches = ceil(static_cast<double>(w.num_samples) / static_cast<double>(w.batch_size));
  const double per_batch = alpha * w.model_layers * w.seq_len * w.batch_size + beta * w.model_layers;
  return batches * per_batch * w.extra_model_factor;
}

// cost_model.maxmin_allocate (cost_model.py:48-87); caps/demands validated by caller.
void maxmin(const double* caps, const double* demands, int n, double capacity, double* out) {
  std::vector<double> eff(n);
  std::vector<int> active(n);
  for (int i = 0; i < n; ++i) {
    eff[i] = std::min(caps[i], demands[i]);
    out[i] = 0.0;
    active[i] = i;
  }
  double remaining = capacity, level = 0.0;
  while (!active.empty() && remaining > 1e-12) {
    double headroom = eff[active[0]] - level;
    for (size_t j = 1; j < active.size(); ++j) headroom = std::min(headroom, eff[active[j]] - level);
    const double step = remaining / static_cast<double>(active.size());
    if (headroom <= step) {
      level += headroom;
      remaining -= headroom * static_cast<double>(active.size());
      for (int i : active) out[i] = std::min(eff[i], level);
      std::vector<int> keep;
      for (int i : active)
        if (eff[i] - level > 1e-12) keep.push_back(i);
      active.swap(keep);
    } else {
      level += step;
      for (int i : active) out[i] = level;
      remaining = 0.0;
    }
  }
}

struct Timer {
  double t;
  int rank;
  int id_rank;  // position of the client id in byte order
  int client;
  int executor;
};
struct TimerLater {
  bool operator()(const Timer& a, const Timer& b) const {
    if (a.t != b.t) return a.t > b.t;
    if (a.rank != b.rank) return a.rank > b.rank;
    if (a.id_rank != b.id_rank) return a.id_rank > b.id_rank;
    return a.executor > b.executor;
  }
};

}  // namespace

struct fedhc_des {
  // ---- inputs of the current round ----
  int n = 0;
  fedhc_des_config cfg{};
  std::vector<int> client_of_part;  // participant -> fleet index
  std::vector<int> id_rank;         // participant -> rank of its id in byte order
  std::vector<double> budget;       // participant -> float(resource_budget)
  std::vector<double> work;         // participant -> work units
  const fedhc_des_client* clients = nullptr;

  // ---- executor manager ----
  std::vector<int> slot_life, slot_client;
  std::vector<double> slot_budget;
  std::vector<double> running_budgets;  // SchedulerState.running_budgets
  int planned = 0;
  std::deque<int> avail;
  // pending participants: arrival-order list and (budget, id)-sorted list
  std::vector<int> arr_next, arr_prev, srt_next, srt_prev;
  int arr_head = -1, srt_head = -1, srt_tail = -1, n_pending = 0;
  std::vector<char> is_pending, launched;

  // ---- engine ----
  std::vector<int> executor_of;
  std::vector<std::vector<double>> phase_work;
  std::vector<int> phase_idx;
  std::vector<double> assigned;
  std::vector<int> running;  // insertion order
  std::priority_queue<Timer, std::vector<Timer>, TimerLater> timers;

  // ---- trace ----
  std::vector<fedhc_des_event> events;
  std::vector<int32_t> alloc_client;
  std::vector<double> alloc_share;
  std::vector<double> par_t;
  std::vector<int32_t> par_n;
  std::string error;

  void emit(double t, int kind, int client, int executor, int aux, double b) {
    fedhc_des_event e{};
    e.t = t;
    e.kind = kind;
    e.client = client;
    e.executor = executor;
    e.aux = aux;
    e.budget = b;
    events.push_back(e);
  }

  double running_total() const {
    PySum s;
    for (double b : running_budgets) s.add(b);
    return s.value();
  }

  double occupied_budget() const {
    PySum s;
    for (size_t i = 0; i < slot_life.size(); ++i)
      if (slot_life[i] == kLaunching || slot_life[i] == kRunning) s.add(slot_budget[i]);
    return s.value();
  }

  void issue(int instr, int ex, double now) { emit(now, FEDHC_EV_INSTRUCTION, slot_client[ex], ex, instr, 0.0); }

  // scheduler._try_accept (scheduler.py:40-52)
  bool try_accept(int p, std::vector<std::pair<int, int>>& acc) {
    if (budget[p] + running_total() <= cfg.theta + kEpsSched && !avail.empty()) {
      const int ex = avail.front();
      avail.pop_front();
      running_budgets.push_back(budget[p]);
      ++planned;
      acc.emplace_back(p, ex);
      return true;
    }
    return false;
  }

  bool guard() const { return planned < n_target && running_total() < cfg.theta - kEpsSched; }
  int n_target = 0;

  // scheduler.schedule_resource_aware (scheduler.py:55-98) over the sorted list
  void sched_ra(std::vector<std::pair<int, int>>& acc) {
    int left = srt_head, right = srt_tail;
    int left_pos = 0, right_pos = n_pending - 1;  // positions in the current sorted order
    bool right_enabled = true;
    while (guard()) {
      if (left_pos > right_pos) break;
      if (!try_accept(left, acc)) return;
      left = srt_next[left];
      ++left_pos;
      if (!guard()) return;
      if (left_pos > right_pos) break;
      if (right_enabled) {
        if (!try_accept(right, acc))
          right_enabled = false;
        else {
          right = srt_prev[right];
          --right_pos;
        }
      }
    }
  }

  // scheduler.schedule_greedy (scheduler.py:101-124) over arrival order
  void sched_greedy(std::vector<std::pair<int, int>>& acc) {
    int cur = arr_head;
    while (cur != -1 && planned < n_target && running_total() < cfg.theta - kEpsSched) {
      if (!try_accept(cur, acc)) break;
      cur = arr_next[cur];
    }
  }

  void unlink(int p) {
    if (arr_prev[p] != -1) arr_next[arr_prev[p]] = arr_next[p]; else arr_head = arr_next[p];
    if (arr_next[p] != -1) arr_prev[arr_next[p]] = arr_prev[p];
    if (srt_prev[p] != -1) srt_next[srt_prev[p]] = srt_next[p]; else srt_head = srt_next[p];
    if (srt_next[p] != -1) srt_prev[srt_next[p]] = srt_prev[p]; else srt_tail = srt_prev[p];
    is_pending[p] = 0;
    --n_pending;
  }

  // ExecutorManager._schedule (executor_manager.py:201-238); returns launches
  bool schedule(double now, int only, std::vector<std::pair<int, int>>& launches) {
    launches.clear();
    if (n_pending == 0) return true;
    std::vector<std::pair<int, int>> acc;
    if (only < 0) {
      if (cfg.scheduler == 0) sched_ra(acc); else sched_greedy(acc);
    } else {
      auto it = std::find(avail.begin(), avail.end(), only);
      if (it == avail.end()) return true;
      std::deque<int> saved;
      saved.swap(avail);
      avail.push_back(only);
      if (cfg.scheduler == 0) sched_ra(acc); else sched_greedy(acc);
      std::deque<int> leftover;
      leftover.swap(avail);
      saved.erase(std::find(saved.begin(), saved.end(), only));
      for (int e : leftover) saved.push_back(e);
      avail.swap(saved);
    }
    for (auto& pe : acc) unlink(pe.first);
    for (auto& pe : acc) {
      const int p = pe.first, ex = pe.second;
      if (slot_life[ex] != kIdle || launched[p]) {
        error = "internal: relaunch or busy slot";
        return false;
      }
      launched[p] = 1;
      slot_life[ex] = kLaunching;
      slot_client[ex] = p;
      slot_budget[ex] = budget[p];
      issue(kInLaunch, ex, now);
      launches.push_back(pe);
    }
    return true;
  }

  int slot_of(int p) const {
    for (size_t i = 0; i < slot_life.size(); ++i)
      if (slot_client[i] == p && slot_life[i] != kIdle) return static_cast<int>(i);
    return -1;
  }

  // ExecutorManager.on_request (executor_manager.py:132-149)
  void on_request(int p, int kind, double now) {
    const int ex = slot_of(p);
    if (ex < 0) return;
    if (kind == 0) {  // REGISTER
      if (slot_life[ex] != kLaunching) return;
      slot_life[ex] = kRunning;
      issue(kInStart, ex, now);
    } else if (kind == 1) {  // TRAINING_COMPLETE
      issue(kInUpload, ex, now);
    } else {  // MODEL_UPLOADED
      slot_life[ex] = kTerminating;
      issue(kInTerminate, ex, now);
    }
  }

  void push_timer(double t, int kind, int p, int ex) { timers.push(Timer{t, kind, id_rank[p], p, ex}); }

  void handle_launches(const std::vector<std::pair<int, int>>& launches, double now) {
    for (auto& pe : launches) {
      executor_of[pe.first] = pe.second;
      emit(now, FEDHC_EV_LAUNCHED, pe.first, pe.second, 0, budget[pe.first]);
      push_timer(now + cfg.launch_latency, kStart, pe.first, pe.second);
    }
  }

  void training_complete(int p, double now) {
    const int ex = executor_of[p];
    emit(now, FEDHC_EV_TRAINED, p, ex, 0, budget[p]);
    on_request(p, 1, now);
    push_timer(now + cfg.upload_latency, kUploadDone, p, ex);
  }

  bool handle_timer(int kind, int p, int ex, double now) {
    if (kind == kStart) {
      on_request(p, 0, now);
      if (work[p] <= kEpsWork) {
        training_complete(p, now);
        return true;
      }
      const fedhc_des_client& c = clients[client_of_part[p]];
      phase_work[p].resize(c.n_phases);
      for (int i = 0; i < c.n_phases; ++i) phase_work[p][i] = c.phase_frac[i] * work[p];
      phase_idx[p] = 0;
      assigned[p] = 0.0;
      running.push_back(p);
    } else if (kind == kUploadDone) {
      emit(now, FEDHC_EV_UPLOADED, p, ex, 0, budget[p]);
      on_request(p, 2, now);
      push_timer(now + cfg.terminate_latency, kSlotFree, p, ex);
    } else {
      emit(now, FEDHC_EV_SLOT_FREED, p, ex, 0, 0.0);
      // ExecutorManager.on_slot_freed (executor_manager.py:151-163)
      auto it = std::find(running_budgets.begin(), running_budgets.end(), slot_budget[ex]);
      if (it != running_budgets.end()) running_budgets.erase(it);
      slot_life[ex] = kIdle;
      slot_client[ex] = -1;
      slot_budget[ex] = 0.0;
      avail.push_back(ex);
      std::vector<std::pair<int, int>> launches;
      if (!schedule(now, cfg.dynamic_parallelism ? -1 : ex, launches)) return false;
      handle_launches(launches, now);
    }
    return true;
  }

  struct Due {
    int rank, id_rank, kind, p, ex;  // kind: 0..4 timer kinds, 9 = work_done
  };

  bool drain(double now) {
    for (;;) {
      std::vector<Due> due;
      while (!timers.empty() && timers.top().t <= now + kEpsTime) {
        const Timer tm = timers.top();
        timers.pop();
        due.push_back(Due{tm.rank, tm.id_rank, tm.rank, tm.client, tm.executor});
      }
      for (int p : running) {
        if (phase_work[p][phase_idx[p]] <= kEpsWork) {
          const bool more = phase_idx[p] + 1 < static_cast<int>(phase_work[p].size());
          due.push_back(Due{more ? kPhase : kTrained, id_rank[p], 9, p, executor_of[p]});
        }
      }
      if (due.empty()) return true;
      std::stable_sort(due.begin(), due.end(), [](const Due& a, const Due& b) {
        if (a.rank != b.rank) return a.rank < b.rank;
        return a.id_rank < b.id_rank;
      });
      for (const Due& d : due) {
        if (d.kind == 9) {
          const int p = d.p;
          if (phase_idx[p] + 1 < static_cast<int>(phase_work[p].size())) {
            ++phase_idx[p];
            emit(now, FEDHC_EV_PHASE, p, d.ex, phase_idx[p], 0.0);
          } else {
            running.erase(std::find(running.begin(), running.end(), p));
            training_complete(p, now);
          }
        } else if (!handle_timer(d.kind, d.p, d.ex, now)) {
          return false;
        }
      }
    }
  }

  int run(const fedhc_des_client* cl, const char* const* ids, const int32_t* order, int n_order,
          const fedhc_des_config* c, double t0, int round_index, fedhc_des_report* rep, double* start_out,
          double* end_out) {
    clients = cl;
    cfg = *c;
    n = n_order;
    events.clear();
    alloc_client.clear();
    alloc_share.clear();
    par_t.clear();
    par_n.clear();
    error.clear();
    while (!timers.empty()) timers.pop();
    if (cfg.max_executors < 1) return fedhc::fail(FEDHC_ERR_CONFIG, "max_executors must be >= 1");
    client_of_part.assign(order, order + n);
    budget.resize(n);
    work.resize(n);
    std::vector<std::string> too_big;
    for (int p = 0; p < n; ++p) {
      const fedhc_des_client& w = cl[order[p]];
      budget[p] = static_cast<double>(w.budget);
      if (w.budget > cfg.theta) too_big.push_back(ids[order[p]]);
      work[p] = work_units(w, cfg.alpha, cfg.beta);
    }
    if (!too_big.empty()) {
      std::string m = "clients [";
      for (size_t i = 0; i < too_big.size(); ++i) m += (i ? ", '" : "'") + too_big[i] + "'";
      char buf[64];
      snprintf(buf, sizeof buf, "%.17g", cfg.theta);
      return fedhc::fail(FEDHC_ERR_CONFIG, m + "] have budgets above theta=" + buf + " and can never launch");
    }
    // id ranks (byte order == Python str order for UTF-8)
    std::vector<int> by_id(n);
    for (int p = 0; p < n; ++p) by_id[p] = p;
    std::sort(by_id.begin(), by_id.end(),
              [&](int a, int b) { return strcmp(ids[order[a]], ids[order[b]]) < 0; });
    id_rank.assign(n, 0);
    for (int r = 0; r < n; ++r) id_rank[by_id[r]] = r;
    // manager state (ExecutorManager.__init__ + begin_round)
    const int E = cfg.max_executors;
    slot_life.assign(E, kIdle);
    slot_client.assign(E, -1);
    slot_budget.assign(E, 0.0);
    running_budgets.clear();
    planned = 0;
    avail.clear();
    for (int e = 0; e < E; ++e) avail.push_back(e);
    n_target = n;
    arr_next.assign(n, -1);
    arr_prev.assign(n, -1);
    for (int p = 0; p < n; ++p) {
      arr_prev[p] = p - 1;
      arr_next[p] = p + 1 < n ? p + 1 : -1;
    }
    arr_head = n ? 0 : -1;
    std::vector<int> srt(n);
    for (int p = 0; p < n; ++p) srt[p] = p;
    std::sort(srt.begin(), srt.end(), [&](int a, int b) {
      if (budget[a] != budget[b]) return budget[a] < budget[b];
      return id_rank[a] < id_rank[b];
    });
    srt_next.assign(n, -1);
    srt_prev.assign(n, -1);
    for (int i = 0; i < n; ++i) {
      srt_prev[srt[i]] = i ? srt[i - 1] : -1;
      srt_next[srt[i]] = i + 1 < n ? srt[i + 1] : -1;
    }
    srt_head = n ? srt[0] : -1;
    srt_tail = n ? srt[n - 1] : -1;
    n_pending = n;
    is_pending.assign(n, 1);
    launched.assign(n, 0);
    executor_of.assign(n, -1);
    phase_work.assign(n, {});
    phase_idx.assign(n, 0);
    assigned.assign(n, 0.0);
    running.clear();

    double t = t0;
    // kickoff (executor_manager.py:120-128)
    std::vector<std::pair<int, int>> launches;
    if (cfg.dynamic_parallelism) {
      if (!schedule(t, -1, launches)) return fedhc::fail(FEDHC_ERR_RUNTIME, error);
      handle_launches(launches, t);
    } else {
      std::vector<std::pair<int, int>> all, one;
      std::vector<int> idle;
      for (int e = 0; e < E; ++e)
        if (slot_life[e] == kIdle) idle.push_back(e);
      for (int e : idle) {
        if (!schedule(t, e, one)) return fedhc::fail(FEDHC_ERR_RUNTIME, error);
        all.insert(all.end(), one.begin(), one.end());
      }
      handle_launches(all, t);
    }
    bool have_last = false;
    std::vector<int> last_ids;
    std::vector<double> last_shares;
    std::vector<int> cur;
    std::vector<double> caps, dem, shares;
    for (;;) {
      if (!drain(t)) return fedhc::fail(FEDHC_ERR_RUNTIME, error);
      if (running.empty() && timers.empty()) break;
      cur = running;
      std::sort(cur.begin(), cur.end(), [&](int a, int b) { return id_rank[a] < id_rank[b]; });
      const int m = static_cast<int>(cur.size());
      caps.resize(m);
      dem.resize(m);
      shares.resize(m);
      for (int i = 0; i < m; ++i) {
        const int p = cur[i];
        caps[i] = budget[p];
        dem[i] = clients[client_of_part[p]].phase_demand[phase_idx[p]];
      }
      maxmin(caps.data(), dem.data(), m, kCapacity, shares.data());
      for (int i = 0; i < m; ++i) assigned[cur[i]] = shares[i];
      const bool same = have_last && last_ids == cur && last_shares == shares;
      if (!same) {
        fedhc_des_event e{};
        e.t = t;
        e.kind = FEDHC_EV_ALLOC;
        e.client = -1;
        e.executor = -1;
        e.alloc_off = static_cast<int64_t>(alloc_client.size());
        e.alloc_len = m;
        for (int i = 0; i < m; ++i) {
          alloc_client.push_back(cur[i]);
          alloc_share.push_back(shares[i]);
        }
        events.push_back(e);
        have_last = true;
        last_ids = cur;
        last_shares = shares;
      }
      if (!(occupied_budget() <= cfg.theta + 1e-6))
        return fedhc::fail(FEDHC_ERR_RUNTIME, "occupied budget exceeds theta");
      double dt_work = INFINITY;
      for (int p : running) dt_work = std::min(dt_work, phase_work[p][phase_idx[p]] / (assigned[p] / kCapacity));
      const double dt_timer = timers.empty() ? INFINITY : timers.top().t - t;
      const double dt = std::min(dt_work, dt_timer);
      if (dt == INFINITY) return fedhc::fail(FEDHC_ERR_RUNTIME, "simulation stalled with work outstanding");
      if (dt > 0) {
        for (int p : running) {
          double& w = phase_work[p][phase_idx[p]];
          w -= assigned[p] / kCapacity * dt;
          if (w < kEpsWork) w = 0.0;
        }
        t += dt;
      }
    }
    if (n_pending) return fedhc::fail(FEDHC_ERR_RUNTIME, "round ended with unlaunched participants");
    if (have_last && !last_ids.empty()) {
      fedhc_des_event e{};
      e.t = t;
      e.kind = FEDHC_EV_ALLOC;
      e.client = -1;
      e.executor = -1;
      e.alloc_off = static_cast<int64_t>(alloc_client.size());
      e.alloc_len = 0;
      events.push_back(e);
    }
    emit(t, FEDHC_EV_ROUND_COMPLETE, -1, -1, round_index, 0.0);
    report(rep, start_out, end_out);
    return FEDHC_OK;
  }

  // metrics.build_round_report (metrics.py:151-167)
  void report(fedhc_des_report* rep, double* start_out, double* end_out) {
    const double start = events.front().t;
    double end = 0.0;
    bool any_up = false;
    int completed = 0;
    for (const auto& e : events)
      if (e.kind == FEDHC_EV_UPLOADED) {
        end = any_up ? std::max(end, e.t) : e.t;
        any_up = true;
        ++completed;
      }
    if (!any_up)
      for (const auto& e : events)
        if (e.kind == FEDHC_EV_ROUND_COMPLETE) {
          end = e.t;
          break;
        }
    // vacancy over the budget step function
    double vac = 0.0, prev_t = start, total = 0.0;
    int count = 0;
    par_t.push_back(start);
    par_n.push_back(0);
    for (const auto& e : events) {
      if (e.kind == FEDHC_EV_LAUNCHED || e.kind == FEDHC_EV_UPLOADED) {
        vac += std::max(0.0, kCapacity - total) * (e.t - prev_t);
        prev_t = e.t;
        if (e.kind == FEDHC_EV_LAUNCHED) {
          total += e.budget;
          ++count;
        } else {
          total -= e.budget;
          --count;
        }
        par_t.push_back(e.t);
        par_n.push_back(count);
      }
    }
    vac += std::max(0.0, kCapacity - total) * (end - prev_t);
    par_t.push_back(end);
    par_n.push_back(count);
    const double makespan = end - start;
    double util = 0.0;
    if (makespan > 0) {
      double area = 0.0, pt = start, ptot = 0.0;
      for (const auto& e : events) {
        if (e.kind != FEDHC_EV_ALLOC) continue;
        area += ptot * (e.t - pt);
        pt = e.t;
        PySum s;
        for (int i = 0; i < e.alloc_len; ++i) s.add(alloc_share[e.alloc_off + i]);
        ptot = s.value();
      }
      area += ptot * (end - pt);
      util = area / (kCapacity * makespan);
    }
    rep->makespan = makespan;
    rep->utilization = util;
    rep->vacancy_area = vac;
    rep->throughput = (completed == 0 || end <= start) ? 0.0 : completed / (end - start);
    rep->degenerate = makespan <= 0;
    rep->n_events = static_cast<int32_t>(events.size());
    rep->n_alloc_pairs = static_cast<int64_t>(alloc_client.size());
    if (start_out || end_out) {
      for (int p = 0; p < n; ++p) {
        if (start_out) start_out[p] = NAN;
        if (end_out) end_out[p] = NAN;
      }
      for (const auto& e : events) {
        if (e.kind == FEDHC_EV_LAUNCHED && start_out) start_out[e.client] = e.t;
        if (e.kind == FEDHC_EV_UPLOADED && end_out) end_out[e.client] = e.t;
      }
    }
  }
};

extern "C" fedhc_des* fedhc_des_create(void) { return new fedhc_des(); }
extern "C" void fedhc_des_destroy(fedhc_des* sim) { delete sim; }

extern "C" int fedhc_des_run_round(fedhc_des* sim, const fedhc_des_client* clients, const char* const* client_ids,
                                   const int32_t* order, int n_order, const fedhc_des_config* cfg, double t0,
                                   int round_index, int record_trace, double* start_out, double* end_out,
                                   fedhc_des_report* report) {
  (void)record_trace;  // the trace is always kept (the report is computed from it)
  if (!sim || !cfg || !report || (n_order > 0 && (!clients || !client_ids || !order)))
    return fedhc::fail(FEDHC_ERR_VALUE, "des: null argument");
  return sim->run(clients, client_ids, order, n_order, cfg, t0, round_index, report, start_out, end_out);
}

extern "C" int fedhc_des_trace(const fedhc_des* sim, const fedhc_des_event** events, const int32_t** alloc_client,
                               const double** alloc_share, const double** par_t, const int32_t** par_n,
                               int* n_par) {
  if (!sim) return fedhc::fail(FEDHC_ERR_VALUE, "des: null handle");
  *events = sim->events.data();
  *alloc_client = sim->alloc_client.data();
  *alloc_share = sim->alloc_share.data();
  *par_t = sim->par_t.data();
  *par_n = sim->par_n.data();
  *n_par = static_cast<int>(sim->par_t.size());
  return FEDHC_OK;
}

extern "C" double fedhc_work_units(int num_samples, int batch_size, int model_layers, int seq_len,
                                   double extra_model_factor, double alpha, double beta) {
  fedhc_des_client c{};
  c.num_samples = num_samples;
  c.batch_size = batch_size;
  c.model_layers = model_layers;
  c.seq_len = seq_len;
  c.extra_model_factor = extra_model_factor;
  return work_units(c, alpha, beta);
}

extern "C" int fedhc_maxmin_allocate(const double* caps, const double* demands, int n, double capacity,
                                     double* alloc_out) {
  for (int i = 0; i < n; ++i) {
    if (!(caps[i] > 0 && caps[i] <= 100)) return fedhc::fail(FEDHC_ERR_CONFIG, "cap outside (0,100]");
    if (!(demands[i] > 0 && demands[i] <= 100)) return fedhc::fail(FEDHC_ERR_CONFIG, "demand outside (0,100]");
  }
  maxmin(caps, demands, n, capacity, alloc_out);
  return FEDHC_OK;
}
