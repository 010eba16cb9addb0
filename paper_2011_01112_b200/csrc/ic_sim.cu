// ic_sim.cu — NEXT-4: event-driven simulation of many RTDeepIoT edge servers
// (include/ic_sim.h).  Host code: each server is a small event machine; servers are
// advanced in lockstep rounds, and every round the planner's DP for all servers that
// reached a scheduling point runs as ONE batched GPU solve (ic_sched_solve_batch_host).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../gen/ic_gen_core.h"
#include "../../include/ic_sched.h"
#include "../../include/ic_sim.h"

namespace {

constexpr int64_t NEVER = INT64_MAX / 4;
constexpr int KMAX = 15;

struct Req {
  int64_t arrive, dabs;
  int client, s, planned;
  int64_t best;  // outcome so far: confidence of the last stage done by dabs
  int32_t w[KMAX], R[KMAX];
};

struct Server {
  int64_t now = 0, busy_until = NEVER;
  int64_t plan_until = 0;  // cost model: no stage starts before the plan is ready
  int64_t plan_carry = 0;  // table cells not yet charged (planning time accrues in whole ticks)
  int running = -1;  // index into reqs of the stage in flight
  bool dirty = false;
  int rr_last = -1;
  std::vector<Req> reqs;  // pending (not yet answered)
  std::vector<int64_t> client_next;
  std::vector<int> client_left, client_seq;
  bool done = false;
};

struct Sim {
  ic_sim_config c;
  int L;
  std::vector<Server> sv;
  int64_t requests = 0, misses = 0, stages = 0, plans = 0, rounds = 0, conf = 0;
  int64_t plan_ticks = 0, busy_ticks = 0;
};

// A request's trace: deadline, stage WCETs, true confidence curve (the generator's recipe).
Req make_request(const Sim& S, int server, int client, int seq, int64_t t) {
  const ic_sim_config& c = S.c;
  const uint64_t gid = ((uint64_t)server << 32) | ((uint64_t)client << 20) | (uint64_t)seq;
  uint32_t x[4], y[4];
  ic_gen_draw(c.seed, gid, 0u, 0u, x);
  Req q{};
  q.arrive = t;
  q.client = client;
  q.s = 0;
  q.planned = S.L;
  q.best = 0;
  const int64_t D = ic_gen_uniform(x[0], c.d_lo, c.d_hi);
  const int easy = (int)(x[1] >> 31);
  const int64_t a0 = easy ? ic_gen_uniform(x[2], 800000, 990000) : ic_gen_uniform(x[2], 100000, 600000);
  const uint32_t rho = (uint32_t)ic_gen_uniform(x[3], 19661, 52429);
  int64_t resid = 1000000 - a0;
  for (int j = 0; j < S.L; ++j) {
    if ((j & 3) == 0) ic_gen_draw(c.seed, gid, 1u, 1u + (uint32_t)(j >> 2), y);
    const uint64_t f = (uint64_t)ic_gen_mulhi32(y[j & 3], 6554u);
    const int64_t w = std::max<int64_t>(1, ((int64_t)c.wcet_base * (65536 + (int64_t)f) + 32768) >> 16);
    q.w[j] = (int32_t)w;
    if (j == 0) {
      q.R[0] = (int32_t)a0;
    } else {
      const int64_t nr = (resid * rho) >> 16;
      q.R[j] = q.R[j - 1] + (int32_t)(resid - nr);
      resid = nr;
    }
  }
  // The planner runs only at GPU-idle instants, so no stage can block the plan it makes:
  // the raw deadline is exact there and the P:L73-75 one-stage adjustment is not needed.
  q.dabs = t + D;
  return q;
}

// Open loop: the gap to a client's next request, uniform in [period/2, 3*period/2].
int64_t open_gap(const Sim& S, int server, int client, int seq) {
  uint32_t x[4];
  ic_gen_draw(S.c.seed, ((uint64_t)server << 32) | ((uint64_t)client << 20) | (uint64_t)seq, 3u, 0u, x);
  const int64_t p = S.c.period;
  return std::max<int64_t>(1, ic_gen_uniform(x[0], p / 2, p + p / 2));
}

void answer(Sim& S, Server& v, int idx, int64_t t) {
  Req& q = v.reqs[idx];
  S.requests++;
  S.conf += q.best;
  if (q.best == 0) S.misses++;
  const int c = q.client;
  if (S.c.period == 0 && v.client_left[c] > 0) v.client_next[c] = t + S.c.think;  // closed loop
  if (v.running > idx) v.running--;
  if (v.rr_last >= idx) v.rr_last--;
  v.reqs.erase(v.reqs.begin() + idx);
}

// Advance a server until it needs a plan (planner) or runs out of events.
// Returns true if it stopped at a scheduling point that needs a DP plan.
bool advance(Sim& S, Server& v) {
  const int pol = S.c.policy;
  for (;;) {
    // Answer requests past their deadline, with every stage done, or — started ones —
    // done with their planned stages.  An unstarted request the plan dropped stays pending
    // until its deadline: later re-plans may admit it.
    for (int i = (int)v.reqs.size() - 1; i >= 0; --i) {
      if (i == v.running) continue;
      const Req& q = v.reqs[i];
      if (q.s >= S.L || q.dabs <= v.now || (q.s > 0 && q.s >= q.planned)) answer(S, v, i, v.now);
    }
    if (v.running < 0 && v.now >= v.plan_until) {
      if (!v.reqs.empty()) {
        if (pol == IC_SIM_PLANNER && v.dirty) return true;
        int pick = -1;
        for (int i = 0; i < (int)v.reqs.size(); ++i) {
          const Req& q = v.reqs[i];
          if (q.s >= q.planned) continue;
          if (pick < 0) { pick = i; continue; }
          const Req& p = v.reqs[pick];
          bool better;
          if (pol == IC_SIM_LCF) {
            const int64_t cq = q.s ? q.R[q.s - 1] : -1, cp = p.s ? p.R[p.s - 1] : -1;
            better = cq < cp || (cq == cp && (q.dabs < p.dabs || (q.dabs == p.dabs && q.arrive < p.arrive)));
          } else if (pol == IC_SIM_RR) {
            better = false;  // handled below
          } else {
            better = q.dabs < p.dabs || (q.dabs == p.dabs && q.arrive < p.arrive);
          }
          if (better) pick = i;
        }
        if (pol == IC_SIM_RR) {
          pick = -1;
          const int n = (int)v.reqs.size();
          for (int k = 1; k <= n; ++k) {
            const int i = (v.rr_last + k) % n;
            if (v.reqs[i].s < v.reqs[i].planned) { pick = i; break; }
          }
          if (pick >= 0) v.rr_last = pick;
        }
        if (pick >= 0) {
          v.running = pick;
          v.busy_until = v.now + v.reqs[pick].w[v.reqs[pick].s];
          S.busy_ticks += v.reqs[pick].w[v.reqs[pick].s];
          S.stages++;
        }
      }
    }
    // next event: an arrival, the completion of the stage in flight, or a waiting request's
    // deadline (arrivals first, then the completion, at equal times)
    int64_t t_arr = NEVER;
    for (size_t c = 0; c < v.client_next.size(); ++c)
      if (v.client_left[c] > 0) t_arr = std::min(t_arr, v.client_next[c]);
    for (int i = 0; i < (int)v.reqs.size(); ++i)
      if (i != v.running) t_arr = std::min(t_arr, v.reqs[i].dabs);
    const int64_t t_done = v.running >= 0 ? v.busy_until : v.plan_until > v.now ? v.plan_until : NEVER;
    const int64_t t = std::min(t_arr, t_done);
    if (t >= NEVER) {
      v.done = true;
      return false;
    }
    v.now = t;
    for (size_t c = 0; c < v.client_next.size(); ++c) {
      if (v.client_left[c] > 0 && v.client_next[c] == t) {
        v.reqs.push_back(make_request(S, (int)(&v - &S.sv[0]), (int)c, v.client_seq[c]++, t));
        v.client_left[c]--;
        v.client_next[c] = S.c.period ? t + open_gap(S, (int)(&v - &S.sv[0]), (int)c, v.client_seq[c]) : NEVER;
        v.dirty = true;
      }
    }
    if (v.running >= 0 && v.busy_until == t) {
      Req& q = v.reqs[v.running];
      q.s++;
      if (t <= q.dabs) q.best = q.R[q.s - 1];  // results after the deadline do not count
      v.running = -1;
      v.busy_until = NEVER;
      v.dirty = true;
    }
  }
}

// The planner's DP instance of a server at a scheduling point (time origin = now, GPU free).
// Returns the size of the paper's reward-indexed table for the instance (the scheduler cost
// model): rows in EDF order, row i spanning Qpre_i + 1 reward columns with S_i + 2 options.
int64_t build_instance(const Sim& S, const Server& v, std::vector<int64_t>& tb, std::vector<int32_t>& rel,
                       std::vector<int32_t>& dl, std::vector<int32_t>& mw, std::vector<uint8_t>& no,
                       std::vector<int32_t>& ow, std::vector<uint32_t>& mc, std::vector<int32_t>& og) {
  const int st = S.L - 1;
  std::vector<std::pair<int64_t, int64_t>> rows;  // (deadline, max quantised reward) per task
  for (const Req& q : v.reqs) {
    // predicted cumulative confidence after each stage (completed stages are sunk)
    int64_t pred[KMAX];
    for (int j = 0; j < S.L; ++j) {
      if (S.c.utility == IC_SIM_UTIL_ORACLE || j < q.s) {
        pred[j] = q.R[j];
      } else {
        const int64_t prev = j == 0 ? -1 : pred[j - 1];
        pred[j] = j == 0 ? S.c.prior_micro : prev + (1000000 - prev) / 2;  // Exp
      }
    }
    // Completed stages are sunk: the DP values each task relative to its current
    // confidence `base`.  Carrying base mod Delta into the mandatory value makes the DP's
    // floor(R/Delta) equal floor(pred/Delta) - floor(base/Delta), i.e. the paper's objective
    // (quantised total confidence, Eq. 1) minus a per-plan constant.
    const int64_t base = q.s ? q.R[q.s - 1] : 0;
    const int64_t carry = base % (int64_t)S.c.delta_micro;
    rel.push_back(0);
    dl.push_back((int32_t)std::max<int64_t>(-1, std::min<int64_t>(q.dabs - v.now, (int64_t)INT32_MAX / 2)));
    mw.push_back(q.w[q.s]);
    no.push_back((uint8_t)(S.L - 1 - q.s));
    mc.push_back((uint32_t)std::max<int64_t>(0, pred[q.s] - base + carry));
    for (int k = 0; k < st; ++k) {
      const int j = q.s + 1 + k;
      ow.push_back(j < S.L ? q.w[j] : 0);
      og.push_back(j < S.L ? (int32_t)(pred[j] - pred[j - 1]) : 0);
    }
    int64_t qm = 0;
    for (int j = q.s; j < S.L; ++j) qm = std::max<int64_t>(qm, (pred[j] - base + carry) / S.c.delta_micro);
    rows.push_back({q.dabs, qm * 16 + (S.L - q.s)});
  }
  tb.push_back(tb.back() + (int64_t)v.reqs.size());
  std::sort(rows.begin(), rows.end());
  int64_t qpre = 0, cells = 0;
  for (const auto& r : rows) {
    qpre += r.second >> 4;
    cells += (qpre + 1) * ((r.second & 15) + 1);
  }
  return cells;
}

}  // namespace

extern "C" int ic_sim_run(const ic_sim_config* cfg, ic_sim_result* out) { return ic_sim_run_dump(cfg, out, nullptr); }

extern "C" int ic_sim_run_dump(const ic_sim_config* cfg, ic_sim_result* out, ic_sim_dump* dump) {
  if (!cfg || !out) return -1;
  if (dump) {
    if (dump->cap_instances < 0 || dump->cap_tasks < 0 || !dump->task_begin || !dump->release || !dump->deadline ||
        !dump->mand_wcet || !dump->n_opt || !dump->mand_conf || !dump->kept || !dump->start || !dump->finish ||
        !dump->q_total || !dump->conf_micro || !dump->makespan || !dump->status ||
        (cfg->n_opt > 0 && (!dump->opt_wcet || !dump->opt_gain)))
      return -1;
    dump->n_instances = dump->n_tasks = 0;
    dump->task_begin[0] = 0;
  }
  const ic_sim_config c = *cfg;
  if (c.servers < 1 || c.clients < 1 || c.requests_per_client < 1 || c.n_opt < 0 || c.n_opt > KMAX - 1 ||
      c.wcet_base < 1 || c.d_lo < 1 || c.d_hi < c.d_lo || c.think < 1 || c.period < 0 || c.policy < 0 || c.policy > 3 ||
      c.plan_cells_per_tick < 0 ||
      (c.policy == IC_SIM_PLANNER && c.delta_micro == 0))
    return -1;
  const auto t0 = std::chrono::steady_clock::now();
  Sim S;
  S.c = c;
  S.L = 1 + c.n_opt;
  S.sv.resize(c.servers);
  for (int i = 0; i < c.servers; ++i) {
    Server& v = S.sv[i];
    v.client_next.assign(c.clients, 0);
    for (int k = 0; k < c.clients; ++k) {  // staggered first arrivals in [0, d_hi)
      uint32_t x[4];
      ic_gen_draw(c.seed, ((uint64_t)i << 32) | ((uint64_t)k << 20) | 0xFFFFFu, 2u, 0u, x);
      v.client_next[k] = ic_gen_uniform(x[0], 0, c.d_hi - 1);
    }
    v.client_left.assign(c.clients, c.requests_per_client);
    v.client_seq.assign(c.clients, 0);
  }
  ic_sched* h = nullptr;
  double gpu_s = 0;
  if (c.policy == IC_SIM_PLANNER) {
    // horizon: every adjusted deadline relative to a scheduling point is < d_hi
    // pending requests: one per client (closed loop), or every arrival within the last
    // d_hi ticks (open loop, gaps >= period/2)
    const int64_t per = c.period ? (int64_t)c.clients * ((int64_t)c.d_hi / std::max(1, c.period / 2) + 1)
                                 : (int64_t)c.clients;
    ic_sched_config sc{c.device, IC_DROP_ALLOWED, c.delta_micro, 0, (int32_t)std::min<int64_t>(per, 4096),
                       c.n_opt, c.d_hi + 1};
    const int rc = ic_sched_create(&sc, &h);
    if (rc != IC_OK) return rc == IC_ERR_CUDA ? -3 : -1;
  }
  std::vector<int> need;
  std::vector<int64_t> tb;
  std::vector<int32_t> rel, dl, mw, ow, og, st, fi, ms;
  std::vector<uint8_t> no, status;
  std::vector<uint32_t> mc;
  std::vector<int8_t> kept;
  std::vector<int64_t> qt, cm;
  std::vector<double> ct;
  for (;;) {
    need.clear();
    bool any = false;
    for (int i = 0; i < c.servers; ++i) {
      Server& v = S.sv[i];
      if (v.done) continue;
      any = true;
      if (advance(S, v)) need.push_back(i);
    }
    if (!any) break;
    if (need.empty()) continue;
    S.rounds++;
    tb.assign(1, 0);
    rel.clear(); dl.clear(); mw.clear(); no.clear(); ow.clear(); mc.clear(); og.clear();
    std::vector<int64_t> cells;
    for (int i : need) cells.push_back(build_instance(S, S.sv[i], tb, rel, dl, mw, no, ow, mc, og));
    const int64_t B = (int64_t)need.size(), T = tb.back();
    kept.resize(T); st.resize(T); fi.resize(T);
    qt.resize(B); cm.resize(B); ct.resize(B); ms.resize(B); status.resize(B);
    ic_batch_in in = {B, tb.data(), rel.data(), dl.data(), mw.data(), no.data(),
                      ow.empty() ? nullptr : ow.data(), mc.data(), og.empty() ? nullptr : og.data()};
    ic_batch_out o = {kept.data(), st.data(), fi.data(), qt.data(), cm.data(), ct.data(), ms.data(), status.data(),
                      nullptr};
    const auto g0 = std::chrono::steady_clock::now();
    const int rc = ic_sched_solve_batch_host(h, &in, &o, nullptr);
    gpu_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - g0).count();
    if (rc != IC_OK) {
      ic_sched_destroy(h);
      return -3;
    }
    S.plans += B;
    if (dump && dump->n_instances + B <= dump->cap_instances && dump->n_tasks + T <= dump->cap_tasks) {
      const int64_t i0 = dump->n_instances, t0 = dump->n_tasks, so = c.n_opt;
      for (int64_t b = 0; b < B; ++b) {
        dump->task_begin[i0 + b + 1] = t0 + tb[b + 1];
        dump->q_total[i0 + b] = qt[b];
        dump->conf_micro[i0 + b] = cm[b];
        dump->makespan[i0 + b] = ms[b];
        dump->status[i0 + b] = status[b];
      }
      for (int64_t k = 0; k < T; ++k) {
        dump->release[t0 + k] = rel[k];
        dump->deadline[t0 + k] = dl[k];
        dump->mand_wcet[t0 + k] = mw[k];
        dump->n_opt[t0 + k] = no[k];
        dump->mand_conf[t0 + k] = mc[k];
        for (int64_t j = 0; j < so; ++j) {
          dump->opt_wcet[(t0 + k) * so + j] = ow[k * so + j];
          dump->opt_gain[(t0 + k) * so + j] = og[k * so + j];
        }
        dump->kept[t0 + k] = kept[k];
        dump->start[t0 + k] = st[k];
        dump->finish[t0 + k] = fi[k];
      }
      dump->n_instances += B;
      dump->n_tasks += T;
    }
    for (int64_t b = 0; b < B; ++b) {
      Server& v = S.sv[need[b]];
      if (c.plan_cells_per_tick > 0) {  // the plan holds the server before the next stage
        v.plan_carry += cells[b];
        const int64_t cost = v.plan_carry / c.plan_cells_per_tick;
        v.plan_carry -= cost * c.plan_cells_per_tick;
        v.plan_until = v.now + cost;
        S.plan_ticks += cost;
      }
      for (int64_t k = tb[b]; k < tb[b + 1]; ++k) {
        Req& q = v.reqs[k - tb[b]];
        q.planned = kept[k] < 0 ? q.s : q.s + 1 + kept[k];  // DROP: stop here (answer now)
      }
      v.dirty = false;
    }
  }
  if (h) ic_sched_destroy(h);
  ic_sim_result r{};
  r.requests = S.requests;
  r.misses = S.misses;
  r.stages_run = S.stages;
  r.plans = S.plans;
  r.rounds = S.rounds;
  r.conf_micro = S.conf;
  r.accuracy = S.requests ? (double)S.conf / 1e6 / (double)S.requests : 0.0;
  r.miss_rate = S.requests ? (double)S.misses / (double)S.requests : 0.0;
  r.mean_depth = S.requests ? (double)S.stages / (double)S.requests : 0.0;
  r.gpu_seconds = gpu_s;
  r.plan_ticks = S.plan_ticks;
  r.busy_ticks = S.busy_ticks;
  r.sim_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = r;
  return 0;
}
