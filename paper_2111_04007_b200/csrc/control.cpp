// Control plane of the Varuna executor, native C++ (host only, no CUDA).
//
//   vp_varuna_schedule / vp_gpipe_schedule  <- spotpipe generate_*_schedule
//        (/root/reference/pkg/src/spotpipe/scheduler.py:128-284)
//   vp_run_replica                           <- spotpipe engine.run_replica
//        (/root/reference/pkg/src/spotpipe/engine/_kernel.pyx:334-567,
//         semantics of engine/py_kernel.py:41-360)
//   vp_assign_stages / vp_identify_cutpoints <- spotpipe partitioner
//        (/root/reference/pkg/src/spotpipe/partitioner.py:124-374)
//
// All time is integer microseconds; results are bit-identical to the
// reference (tests/test_control_parity.py). The replica policy object
// (ReplicaPolicy) is also what the live per-stage dispatcher drives.

#include "vpipe.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <new>
#include <queue>
#include <vector>

namespace {

constexpr int64_t kB = VP_KIND_BACKWARD;
constexpr int64_t kR = VP_KIND_RECOMPUTE;
constexpr int64_t kF = VP_KIND_FORWARD;

// ---------------------------------------------------------------------------
// Static plan: zero-delay simulation of Varuna's rules.
// ---------------------------------------------------------------------------
struct PlanSim {
  int64_t P, N, tf, tb, tr;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> plan;

  int run() {
    const int64_t last = P - 1;
    plan.assign(P, {});
    std::vector<int64_t> end_at(P, 0), cur_kind(P, -1), cur_mb(P, 0), nf(P, 0), nb(P, 0), hold(P, -1);
    // -1 = not yet known.
    std::vector<int64_t> act(P * N, -1), grad(P * N, -1), due(P * N, -1);
    std::vector<uint8_t> recd(P * N, 0);
    for (int64_t j = 0; j < N; ++j) act[j] = 0;
    std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> times;
    times.push(0);
    auto ready = [](int64_t t, int64_t now) { return t >= 0 && t <= now; };
    while (!times.empty()) {
      const int64_t now = times.top();
      while (!times.empty() && times.top() == now) times.pop();
      for (int64_t k = 0; k < P; ++k) {
        if (cur_kind[k] < 0 || end_at[k] != now) continue;
        const int64_t kind = cur_kind[k], mb = cur_mb[k];
        cur_kind[k] = -1;
        if (kind == kF) {
          ++nf[k];
          if (k < last) act[(k + 1) * N + mb] = now;
        } else if (kind == kR) {
          recd[k * N + mb] = 1;
          hold[k] = mb;
        } else {
          ++nb[k];
          if (k > 0) grad[(k - 1) * N + mb] = now;
        }
      }
      for (int64_t k = 0; k < P; ++k) {
        if (cur_kind[k] >= 0 || nb[k] >= N) continue;
        int64_t kind = -1, mb = 0;
        if (hold[k] >= 0) {
          const int64_t j = hold[k];
          if (!ready(grad[k * N + j], now)) continue;
          kind = kB; mb = j;
        } else {
          const int64_t j = nb[k];
          const int64_t g = grad[k * N + j];
          bool skip = false;
          if (k == last) {
            if (nf[k] > j) { kind = kB; mb = j; }
          } else if (ready(g, now) && recd[k * N + j]) {
            kind = kB; mb = j;
          } else if (nf[k] > j && !recd[k * N + j]) {
            if (ready(g, now)) {
              kind = kR; mb = j;
            } else if (due[k * N + j] >= 0) {
              const int64_t d = due[k * N + j];
              if (now >= d) {
                kind = kR; mb = j;
              } else {
                const int64_t f = nf[k];
                if (f < N && ready(act[k * N + f], now) && now + tf <= d) {
                  kind = kF; mb = f;
                } else {
                  times.push(d);
                  skip = true;
                }
              }
            }
          }
          if (skip) continue;
          if (kind < 0) {
            const int64_t f = nf[k];
            if (f < N && ready(act[k * N + f], now)) { kind = kF; mb = f; }
            else continue;
          }
        }
        const int64_t dur = kind == kF ? tf : (kind == kB ? tb : tr);
        plan[k].push_back({kind, mb});
        cur_kind[k] = kind;
        cur_mb[k] = mb;
        end_at[k] = now + dur;
        times.push(now + dur);
        if (kind == kB) {
          hold[k] = -1;
          if (k > 0) {
            const int64_t d = now + tb - tr;
            due[(k - 1) * N + mb] = d;
            times.push(d > now ? d : now);
          }
        }
      }
    }
    for (int64_t k = 0; k < P; ++k)
      if (nb[k] != N) return VP_ERR_DEADLOCK;
    return VP_OK;
  }
};

int emit_plan(const std::vector<std::vector<std::pair<int64_t, int64_t>>>& plan,
              int64_t capacity, int64_t* kinds, int64_t* mbs, int64_t* offsets) {
  int64_t pos = 0;
  offsets[0] = 0;
  for (size_t k = 0; k < plan.size(); ++k) {
    for (auto& t : plan[k]) {
      if (pos >= capacity) return VP_ERR_CAPACITY;
      kinds[pos] = t.first;
      mbs[pos] = t.second;
      ++pos;
    }
    offsets[k + 1] = pos;
  }
  return VP_OK;
}

// ---------------------------------------------------------------------------
// Replica event kernel.
// ---------------------------------------------------------------------------
struct Event {
  int64_t time, stage;
  bool operator>(const Event& o) const { return time != o.time ? time > o.time : stage > o.stage; }
};

struct ReplicaPolicy {
  // inputs
  int64_t P, N;
  const int64_t *kinds, *mbs, *offsets, *fwd, *bwd, *rec, *act_tx, *grad_tx, *exp_grad, *in_act,
      *work, *cap;
  bool opp, serialize;
  // state
  std::vector<uint8_t> executed;
  std::vector<int64_t> ptr, run_kind, run_mb, busy_until, locked, last_done, n_f, n_b;
  std::vector<int64_t> f_pos, b_pos, b_mb, r_pos;    // [P*N]
  std::vector<int64_t> act_arr, grad_arr, deadline;  // [P*N]
  std::vector<int64_t> act_free, grad_free;
  std::vector<int64_t> stash, sets, peak_stash, peak_sets, peak_mem, last_bwd_end;
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> q;
  vp_replica_out* out;
  static constexpr int64_t kFar = int64_t(1) << 60;

  int init() {
    const int64_t T = offsets[P];
    executed.assign(T, 0);
    ptr.assign(offsets, offsets + P);
    run_kind.assign(P, -1);
    run_mb.assign(P, -1);
    busy_until.assign(P, 0);
    locked.assign(P, -1);
    last_done.assign(P, -1);
    n_f.assign(P, 0);
    n_b.assign(P, 0);
    f_pos.assign(P * N, -1);
    b_pos.assign(P * N, -1);
    b_mb.assign(P * N, -1);
    r_pos.assign(P * N, -1);
    for (int64_t k = 0; k < P; ++k) {
      int64_t cf = 0, cb = 0;
      for (int64_t p = offsets[k]; p < offsets[k + 1]; ++p) {
        const int64_t kd = kinds[p], mb = mbs[p];
        if (mb < 0 || mb >= N) return VP_ERR_ARGS;
        if (kd == kF) {
          if (cf >= N) return VP_ERR_ARGS;
          f_pos[k * N + cf++] = p;
        } else if (kd == kB) {
          if (cb >= N) return VP_ERR_ARGS;
          b_pos[k * N + cb] = p;
          b_mb[k * N + cb++] = mb;
        } else if (kd == kR) {
          r_pos[k * N + mb] = p;
        } else {
          return VP_ERR_ARGS;
        }
      }
    }
    act_arr.assign(P * N, -1);
    grad_arr.assign(P * N, -1);
    deadline.assign(P * N, -1);
    for (int64_t j = 0; j < N; ++j) act_arr[j] = 0;
    act_free.assign(std::max<int64_t>(P - 1, 1), 0);
    grad_free.assign(std::max<int64_t>(P - 1, 1), 0);
    stash.assign(P, 0);
    sets.assign(P, 0);
    peak_stash.assign(P, 0);
    peak_sets.assign(P, 0);
    peak_mem.assign(P, 0);
    last_bwd_end.assign(P, 0);
    for (int64_t k = 0; k < P; ++k) q.push({0, k});
    out->n_tasks = 0;
    out->n_msgs = 0;
    return VP_OK;
  }

  void account(int64_t k) {
    peak_stash[k] = std::max(peak_stash[k], stash[k]);
    peak_sets[k] = std::max(peak_sets[k], sets[k]);
    peak_mem[k] = std::max(peak_mem[k], stash[k] * in_act[k] + sets[k] * work[k]);
  }

  void start(int64_t k, int64_t pos, int64_t now) {
    const int64_t kind = kinds[pos], mb = mbs[pos];
    const int64_t dur = kind == kF ? fwd[k] : (kind == kB ? bwd[k] : rec[k]);
    executed[pos] = 1;
    run_kind[k] = kind;
    run_mb[k] = mb;
    busy_until[k] = now + dur;
    const int64_t i = out->n_tasks++;
    out->task_stage[i] = k;
    out->task_kind[i] = kind;
    out->task_mb[i] = mb;
    out->task_start[i] = now;
    out->task_end[i] = now + dur;
    if (kind == kF) {
      ++n_f[k];
      ++stash[k];
      ++sets[k];
      account(k);
    } else if (kind == kR) {
      ++sets[k];
      account(k);
    } else {
      locked[k] = -1;
      if (k > 0) {
        // Rule 1: the stage below should finish recomputing as this
        // backward's gradient lands (estimated with the mean transfer).
        const int64_t dl = now + dur + exp_grad[k - 1] - rec[k - 1];
        deadline[(k - 1) * N + mb] = dl;
        q.push({dl > now ? dl : now, k - 1});
      }
    }
    q.push({now + dur, k});
  }

  void send(int64_t boundary, int dir, int64_t mb, int64_t now) {
    const int64_t dur = dir == 0 ? act_tx[boundary * N + mb] : grad_tx[boundary * N + mb];
    int64_t& free_at = dir == 0 ? act_free[boundary] : grad_free[boundary];
    int64_t grant = now;
    if (serialize) {
      grant = free_at <= now ? now : free_at;
      free_at = grant + dur;
    }
    const int64_t arrive = grant + dur;
    const int64_t i = out->n_msgs++;
    out->msg_send[i] = now;
    out->msg_grant[i] = grant;
    out->msg_arrive[i] = arrive;
    out->msg_boundary[i] = boundary;
    out->msg_dir[i] = dir;
    out->msg_mb[i] = mb;
    if (dir == 0) {
      act_arr[(boundary + 1) * N + mb] = arrive;
      q.push({arrive, boundary + 1});
    } else {
      grad_arr[boundary * N + mb] = arrive;
      q.push({arrive, boundary});
      const int64_t jit = arrive - rec[boundary];
      q.push({jit > now ? jit : now, boundary});
    }
  }

  void complete(int64_t k, int64_t now) {
    const int64_t kind = run_kind[k], mb = run_mb[k];
    run_kind[k] = -1;
    run_mb[k] = -1;
    last_done[k] = kind;
    if (kind == kF) {
      if (k < P - 1) {
        --sets[k];  // checkpointing: intermediates discarded
        send(k, 0, mb, now);
      }
    } else if (kind == kR) {
      locked[k] = mb;
    } else {
      --sets[k];
      --stash[k];
      ++n_b[k];
      last_bwd_end[k] = now;
      if (k > 0) send(k - 1, 1, mb, now);
    }
  }

  int64_t rec_due_at(int64_t k, int64_t mb, int64_t now) const {
    const int64_t g = grad_arr[k * N + mb];
    if (g >= 0) return g <= now ? now : g - rec[k];
    const int64_t dl = deadline[k * N + mb];
    return dl >= 0 ? dl : kFar;
  }

  bool arrived(int64_t t, int64_t now) const { return t >= 0 && t <= now; }

  void decide(int64_t k, int64_t now) {
    if (run_kind[k] >= 0) return;
    const bool last = (k == P - 1);
    const int64_t j = locked[k];
    if (j >= 0) {
      // Rule 2: only the matching backward may follow a recompute.
      if (last || arrived(grad_arr[k * N + j], now)) start(k, b_pos[k * N + n_b[k]], now);
      return;
    }
    int64_t p = ptr[k];
    const int64_t end = offsets[k + 1];
    while (p < end && executed[p]) ++p;
    ptr[k] = p;
    if (p >= end) return;
    const int64_t kind = kinds[p], mb = mbs[p];
    if (kind == kB) {
      if (last || arrived(grad_arr[k * N + mb], now)) start(k, p, now);
      return;
    }
    if (kind == kF) {
      const bool capped = opp && stash[k] >= cap[k];
      if (!capped && arrived(act_arr[k * N + mb], now)) {
        start(k, p, now);
        return;
      }
      if (!opp) return;
      // Late activation or full stash: the next recompute/backward pair may
      // jump ahead once its recompute is due.
      const int64_t c = n_b[k];
      if (c < N && !last) {
        const int64_t jb = b_mb[k * N + c];
        const int64_t rp = r_pos[k * N + jb];
        if (rp >= 0 && !executed[rp] && n_f[k] > jb && now >= rec_due_at(k, jb, now))
          start(k, rp, now);
      }
      return;
    }
    // Recompute at the head.
    if (!opp || last) {
      start(k, p, now);
      return;
    }
    const int64_t f = n_f[k];
    const bool f_ready = f < N && arrived(act_arr[k * N + f], now) && stash[k] < cap[k];
    if (arrived(grad_arr[k * N + mb], now)) {
      // Running late: pace the backlog with one ready forward per pair.
      if (f_ready && last_done[k] == kB) start(k, f_pos[k * N + f], now);
      else start(k, p, now);
      return;
    }
    const int64_t due = rec_due_at(k, mb, now);
    if (now >= due) {
      start(k, p, now);
      return;
    }
    if (f_ready) {
      if (now + fwd[k] <= due) start(k, f_pos[k * N + f], now);
      return;  // hold the slot for the just-in-time recompute
    }
    start(k, p, now);
  }

  int loop() {
    std::vector<uint8_t> touched(P, 0);
    std::vector<int64_t> touched_list;
    touched_list.reserve(P);
    while (!q.empty()) {
      const int64_t now = q.top().time;
      touched_list.clear();
      while (!q.empty() && q.top().time == now) {
        const int64_t k = q.top().stage;
        q.pop();
        if (run_kind[k] >= 0 && busy_until[k] == now) complete(k, now);
        if (!touched[k]) {
          touched[k] = 1;
          touched_list.push_back(k);
        }
      }
      std::sort(touched_list.begin(), touched_list.end());
      for (int64_t k : touched_list) {
        touched[k] = 0;
        decide(k, now);
      }
    }
    for (int64_t k = 0; k < P; ++k)
      if (n_b[k] != N) return VP_ERR_DEADLOCK;
    int64_t mk = 0;
    for (int64_t i = 0; i < out->n_tasks; ++i) mk = std::max(mk, out->task_end[i]);
    out->makespan = mk;
    for (int64_t k = 0; k < P; ++k) {
      out->last_bwd_end[k] = last_bwd_end[k];
      out->peak_stash[k] = peak_stash[k];
      out->peak_sets[k] = peak_sets[k];
      out->peak_mem[k] = peak_mem[k];
    }
    return VP_OK;
  }
};

// ---------------------------------------------------------------------------
// Partition DPs.
// ---------------------------------------------------------------------------
constexpr double kInf = std::numeric_limits<double>::infinity();

}  // namespace

extern "C" {

int vp_varuna_schedule(int64_t P, int64_t N, int64_t tf, int64_t tb, int64_t tr, int64_t capacity,
                       int64_t* kinds, int64_t* mbs, int64_t* offsets) {
  if (P < 1 || N < 1) return VP_ERR_ARGS;
  if (tf <= 0 || tb <= 0 || tr <= 0) return VP_ERR_ARGS;
  if (!kinds || !mbs || !offsets) return VP_ERR_ARGS;
  try {
    PlanSim sim{P, N, tf, tb, tr, {}};
    int rc = sim.run();
    if (rc != VP_OK) return rc;
    return emit_plan(sim.plan, capacity, kinds, mbs, offsets);
  } catch (const std::bad_alloc&) {
    return VP_ERR_NOMEM;
  }
}

int vp_gpipe_schedule(int64_t P, int64_t N, int64_t capacity, int64_t* kinds, int64_t* mbs,
                      int64_t* offsets) {
  if (P < 1 || N < 1 || !kinds || !mbs || !offsets) return VP_ERR_ARGS;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> plan(P);
  for (int64_t k = 0; k < P; ++k) {
    auto& t = plan[k];
    for (int64_t j = 0; j < N; ++j) t.push_back({kF, j});
    int64_t first = N - 1;
    if (k == P - 1) {
      t.push_back({kB, N - 1});
      first = N - 2;
    }
    for (int64_t j = first; j >= 0; --j) {
      t.push_back({kR, j});
      t.push_back({kB, j});
    }
  }
  return emit_plan(plan, capacity, kinds, mbs, offsets);
}

int vp_run_replica(int64_t n_stages, int64_t n_micro, const int64_t* kinds, const int64_t* mbs,
                   const int64_t* offsets, const int64_t* fwd_us, const int64_t* bwd_us,
                   const int64_t* rec_us, const int64_t* act_tx_us, const int64_t* grad_tx_us,
                   const int64_t* exp_grad_tx_us, const int64_t* in_act_bytes,
                   const int64_t* work_bytes, const int64_t* stash_cap, int opportunistic,
                   int serialize_links, vp_replica_out* out) {
  if (n_stages < 1 || n_micro < 1 || !out) return VP_ERR_ARGS;
  if (n_stages >= 4096) return VP_ERR_ARGS;
  try {
    ReplicaPolicy r;
    r.P = n_stages;
    r.N = n_micro;
    r.kinds = kinds;
    r.mbs = mbs;
    r.offsets = offsets;
    r.fwd = fwd_us;
    r.bwd = bwd_us;
    r.rec = rec_us;
    r.act_tx = act_tx_us;
    r.grad_tx = grad_tx_us;
    r.exp_grad = exp_grad_tx_us;
    r.in_act = in_act_bytes;
    r.work = work_bytes;
    r.cap = stash_cap;
    r.opp = opportunistic != 0;
    r.serialize = serialize_links != 0;
    r.out = out;
    int rc = r.init();
    if (rc != VP_OK) return rc;
    return r.loop();
  } catch (const std::bad_alloc&) {
    return VP_ERR_NOMEM;
  }
}

// Linear partition of K cut-points into P contiguous stages: min-max forward
// time (last stage scaled by last_stage_weight), ties -> minimal total
// boundary activation, then earliest boundaries. boundaries_out[P].
int vp_assign_stages(int64_t K, const int64_t* forward_us, const int64_t* acts, int64_t P,
                     double last_stage_weight, int64_t* boundaries_out) {
  if (P < 1 || K < 1) return VP_ERR_ARGS;
  if (P > K) return VP_ERR_INFEASIBLE;
  try {
    std::vector<int64_t> pre(K + 1, 0);
    for (int64_t i = 0; i < K; ++i) pre[i + 1] = pre[i] + forward_us[i];
    auto seg = [&](int64_t i, int64_t j) { return pre[j + 1] - pre[i]; };
    auto last_cost = [&](int64_t i) { return last_stage_weight * double(seg(i, K - 1)); };
    std::vector<double> mm((P + 1) * (K + 1), kInf);
    auto MM = [&](int64_t j, int64_t i) -> double& { return mm[j * (K + 1) + i]; };
    for (int64_t i = 0; i < K; ++i) MM(1, i) = last_cost(i);
    for (int64_t j = 2; j <= P; ++j)
      for (int64_t i = 0; i < K; ++i) {
        double best = kInf;
        for (int64_t e = i; e < K - 1; ++e) {
          const double s = double(seg(i, e));
          if (s >= best) break;
          const double rest = MM(j - 1, e + 1);
          const double cand = s > rest ? s : rest;
          if (cand < best) best = cand;
        }
        MM(j, i) = best;
      }
    const double best_max = MM(P, 0);
    // Activation sums are integers; keep them exact in int64 with a sentinel.
    const int64_t kBig = std::numeric_limits<int64_t>::max();
    std::vector<int64_t> ma((P + 1) * (K + 1), kBig);
    auto MA = [&](int64_t j, int64_t i) -> int64_t& { return ma[j * (K + 1) + i]; };
    for (int64_t i = 0; i < K; ++i)
      if (last_cost(i) <= best_max) MA(1, i) = 0;
    for (int64_t j = 2; j <= P; ++j)
      for (int64_t i = 0; i < K; ++i) {
        int64_t best = kBig;
        for (int64_t e = i; e < K - 1; ++e) {
          if (double(seg(i, e)) > best_max) break;
          const int64_t rest = MA(j - 1, e + 1);
          if (rest != kBig && acts[e] + rest < best) best = acts[e] + rest;
        }
        MA(j, i) = best;
      }
    int64_t i = 0, nb = 0;
    for (int64_t j = P; j > 1; --j) {
      const int64_t target = MA(j, i);
      for (int64_t e = i; e < K - 1; ++e) {
        if (double(seg(i, e)) > best_max) break;
        const int64_t rest = MA(j - 1, e + 1);
        if (rest != kBig && acts[e] + rest == target) {
          boundaries_out[nb++] = e;
          i = e + 1;
          break;
        }
      }
    }
    boundaries_out[nb++] = K - 1;
    return nb == P ? VP_OK : VP_ERR_INFEASIBLE;
  } catch (const std::bad_alloc&) {
    return VP_ERR_NOMEM;
  }
}

// Cut-point identification over n operations: min-max section compute time
// over unbreakable-aware splits, then (within cap = max(best,
// ceil((1+tol)*total/K))) minimal boundary activation, earliest first.
int vp_identify_cutpoints(int64_t n, const int64_t* compute_us, const int64_t* acts,
                          const uint8_t* breakable, int64_t K, double tolerance,
                          int64_t* boundaries_out) {
  if (K < 1 || n < 1) return VP_ERR_ARGS;
  if (K > n) return VP_ERR_INFEASIBLE;
  try {
    std::vector<int64_t> pre(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + compute_us[i];
    auto seg = [&](int64_t i, int64_t j) { return pre[j + 1] - pre[i]; };
    std::vector<double> mm((K + 1) * (n + 1), kInf);
    auto MM = [&](int64_t j, int64_t i) -> double& { return mm[j * (n + 1) + i]; };
    for (int64_t i = 0; i < n; ++i) MM(1, i) = double(seg(i, n - 1));
    for (int64_t j = 2; j <= K; ++j)
      for (int64_t i = 0; i < n; ++i) {
        double best = kInf;
        for (int64_t e = i; e < n - 1; ++e) {
          if (!breakable[e]) continue;
          const double s = double(seg(i, e));
          if (s >= best) break;
          const double rest = MM(j - 1, e + 1);
          const double cand = s > rest ? s : rest;
          if (cand < best) best = cand;
        }
        MM(j, i) = best;
      }
    if (std::isinf(MM(K, 0))) return VP_ERR_INFEASIBLE;
    const int64_t total = pre[n];
    const int64_t window = int64_t(std::ceil((1.0 + tolerance) * double(total) / double(K)));
    const int64_t cap = std::max(int64_t(MM(K, 0)), window);
    const int64_t kBig = std::numeric_limits<int64_t>::max();
    std::vector<int64_t> ma((K + 1) * (n + 1), kBig);
    auto MA = [&](int64_t j, int64_t i) -> int64_t& { return ma[j * (n + 1) + i]; };
    for (int64_t i = 0; i < n; ++i)
      if (seg(i, n - 1) <= cap) MA(1, i) = 0;
    for (int64_t j = 2; j <= K; ++j)
      for (int64_t i = 0; i < n; ++i) {
        int64_t best = kBig;
        for (int64_t e = i; e < n - 1; ++e) {
          if (seg(i, e) > cap) break;
          if (!breakable[e]) continue;
          const int64_t rest = MA(j - 1, e + 1);
          if (rest != kBig && acts[e] + rest < best) best = acts[e] + rest;
        }
        MA(j, i) = best;
      }
    if (MA(K, 0) == kBig) return VP_ERR_INFEASIBLE;
    int64_t i = 0, nb = 0;
    for (int64_t j = K; j > 1; --j) {
      const int64_t target = MA(j, i);
      for (int64_t e = i; e < n - 1; ++e) {
        if (seg(i, e) > cap) break;
        if (!breakable[e]) continue;
        const int64_t rest = MA(j - 1, e + 1);
        if (rest != kBig && acts[e] + rest == target) {
          boundaries_out[nb++] = e;
          i = e + 1;
          break;
        }
      }
    }
    boundaries_out[nb++] = n - 1;
    return nb == K ? VP_OK : VP_ERR_INFEASIBLE;
  } catch (const std::bad_alloc&) {
    return VP_ERR_NOMEM;
  }
}

const char* vp_version(void) { return "vpipe 0.1.0 (sm_100a)"; }

}  // extern "C"
