// sched.cpp — FaaSwap's node policies as host C++ in libfsw.
//
//   pure policies (policy.h, exported as fsw_policy_* for tests):
//     RRC ........................ PAPER.md:784-790
//     α partition ................ PAPER.md:794-799
//     α auto-configuration ....... Algorithm 2
//     interference-aware placement Algorithm 1, PAPER.md:845-876  (used by fsw_invoke)
//     heaviness-aware LRU eviction PAPER.md:885-897              (used by the weight pool)
//   request scheduler (fsw_sched_*): two priority queues ordered by RRC over
//   the functions of a node, dispatching onto the pool's GPUs through the public fsw_invoke —
//   the scheduler sits above the swap-and-execute runtime and uses only its C-ABI.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <numeric>
#include <thread>
#include <vector>

#include "fsw.h"
#include "policy.h"

namespace fsw {

double rrc(uint64_t n, uint64_t m, double p) { return (p * (double)n - (double)m) / (1.0 - p); }

std::vector<uint8_t> partition_high(const std::vector<double>& rrcs, double alpha) {
    const size_t n = rrcs.size();
    std::vector<uint32_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0u);
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return rrcs[a] < rrcs[b]; });
    // the total is summed in the same (sorted) order as the prefixes, so the last prefix equals it
    // bit for bit and α = 1 puts every function in the high group
    double total = 0.0;
    for (uint32_t i : idx) total += std::max(rrcs[i], 0.0);
    const double budget = alpha * total;
    std::vector<uint8_t> high(n, 0);
    if (alpha >= 1.0) {
        std::fill(high.begin(), high.end(), 1);
        return high;
    }
    double prefix = 0.0;
    for (uint32_t i : idx) {  // k = the largest prefix whose positive part fits the budget
        prefix += std::max(rrcs[i], 0.0);
        if (prefix > budget) break;
        high[i] = 1;
    }
    return high;
}

double alpha_config(double alpha, double last_ratio, double new_ratio, double scalar, double threshold) {
    const double d = new_ratio - last_ratio, th = std::fabs(threshold);
    if (d > th) return std::min(alpha * scalar, 1.0);
    if (d < -th) return alpha / scalar;
    return alpha;
}

Decision schedule(const std::vector<uint8_t>& available, const std::vector<uint8_t>& hosts,
                  const std::vector<int>& neighbor, const std::vector<uint8_t>& loading, const std::vector<float>& link) {
    const int n = (int)available.size();
    Decision d;
    // lines 4-8: resident on an available GPU -> execute there without swapping
    for (int g = 0; g < n; ++g)
        if (hosts[g] && available[g]) {
            d.gpu = g;
            d.kind = 0;
            return d;
        }
    bool any_avail = false, any_host = false;
    for (int g = 0; g < n; ++g) {
        any_avail |= available[g] != 0;
        any_host |= hosts[g] != 0;
    }
    if (!any_avail) return d;  // A = ∅: the request stays queued
    if (any_host) {
        // lines 10-11: GPU pair (g ∈ A, m ∈ M) with the fastest NVLink; ties -> lowest (g, m)
        float best = -1.0f;
        for (int g = 0; g < n; ++g) {
            if (!available[g]) continue;
            for (int s = 0; s < n; ++s) {
                if (!hosts[s] || s == g) continue;
                const float bw = link.empty() ? 1.0f : link[(size_t)g * n + s];
                if (bw <= 0.0f) continue;  // no NVLink path
                if (bw > best) {
                    best = bw;
                    d.gpu = g;
                    d.src = s;
                }
            }
        }
        if (d.gpu >= 0) {
            d.kind = 2;
            return d;
        }
    }
    // lines 13-20: host swap onto a GPU whose PCIe neighbour is not loading, else one whose
    // neighbour loads a light model, else any available GPU (lowest id in each tier)
    for (int tier = 0; tier < 3; ++tier)
        for (int g = 0; g < n; ++g) {
            if (!available[g]) continue;
            const int nb = neighbor.empty() ? -1 : neighbor[g];
            const int ld = nb >= 0 && nb < n ? loading[nb] : 0;
            if ((tier == 0 && ld == 0) || (tier == 1 && ld == 1) || tier == 2) {
                d.gpu = g;
                d.kind = 1;
                return d;
            }
        }
    return d;
}

bool heavy_by_slo(double swap_ms, double resident_ms, double deadline_ms, double queue_budget_ms, double theta) {
    if (deadline_ms <= 0.0) return resident_ms + swap_ms > 1.25 * resident_ms;
    const double slack = deadline_ms - resident_ms - queue_budget_ms;
    return slack <= 0.0 || swap_ms > theta * slack;
}

std::vector<uint32_t> eviction_order(const std::vector<uint8_t>& heavy, const std::vector<uint32_t>& copies,
                                     const std::vector<uint64_t>& last_use, const std::vector<uint8_t>& in_use) {
    std::vector<uint32_t> low, high;
    for (uint32_t i = 0; i < heavy.size(); ++i) {
        if (in_use[i]) continue;
        (heavy[i] && copies[i] <= 1 ? high : low).push_back(i);
    }
    auto lru = [&](uint32_t a, uint32_t b) { return last_use[a] != last_use[b] ? last_use[a] < last_use[b] : a < b; };
    std::sort(low.begin(), low.end(), lru);
    std::sort(high.begin(), high.end(), lru);
    low.insert(low.end(), high.begin(), high.end());
    return low;
}

}  // namespace fsw

using namespace fsw;

// ==========================================================================================
// exported pure policies
// ==========================================================================================
extern "C" fsw_status fsw_policy_rrc(uint64_t n, uint64_t m, double p, double* out) {
    if (!out || !(p > 0.0 && p < 1.0) || m > n) return FSW_EINVAL;
    *out = rrc(n, m, p);
    return FSW_OK;
}

extern "C" fsw_status fsw_policy_partition(const double* rrcs, uint32_t n, double alpha, uint8_t* high) {
    if ((n && (!rrcs || !high)) || !(alpha >= 0.0 && alpha <= 1.0)) return FSW_EINVAL;
    const std::vector<uint8_t> h = partition_high(std::vector<double>(rrcs, rrcs + n), alpha);
    std::copy(h.begin(), h.end(), high);
    return FSW_OK;
}

extern "C" fsw_status fsw_policy_alpha(double alpha, double last_ratio, double new_ratio, double scalar, double threshold,
                                       double* out) {
    if (!out || !(scalar > 1.0)) return FSW_EINVAL;
    *out = alpha_config(alpha, last_ratio, new_ratio, scalar, threshold);
    return FSW_OK;
}

extern "C" fsw_status fsw_policy_schedule(uint32_t n, const uint8_t* available, const uint8_t* hosts, const int32_t* neighbor,
                                          const uint8_t* loading, const float* link, fsw_decision* out) {
    if (!out || !n || !available || !hosts) return FSW_EINVAL;
    std::vector<int> nb;
    if (neighbor) nb.assign(neighbor, neighbor + n);
    std::vector<uint8_t> ld(n, 0);
    if (loading) ld.assign(loading, loading + n);
    std::vector<float> lk;
    if (link) lk.assign(link, link + (size_t)n * n);
    const Decision d = schedule(std::vector<uint8_t>(available, available + n), std::vector<uint8_t>(hosts, hosts + n), nb, ld, lk);
    out->gpu = d.gpu;
    out->kind = (uint32_t)d.kind;
    out->src = d.src;
    return d.gpu < 0 ? FSW_EBUSY : FSW_OK;
}

std::vector<uint32_t> fsw::stripe_deal(const std::vector<int>& unit_node, const std::vector<int>& src_node) {
    const uint32_t n = (uint32_t)src_node.size();
    std::map<int, std::vector<uint32_t>> by_node;
    for (uint32_t j = 0; j < n; ++j)
        if (src_node[j] >= 0) by_node[src_node[j]].push_back(j);
    std::map<int, uint64_t> ctr;
    uint64_t any = 0;
    std::vector<uint32_t> out(unit_node.size(), 0);
    for (size_t u = 0; u < unit_node.size(); ++u) {
        auto it = unit_node[u] >= 0 ? by_node.find(unit_node[u]) : by_node.end();
        if (it == by_node.end()) out[u] = n ? (uint32_t)(any++ % n) : 0;
        else out[u] = it->second[ctr[unit_node[u]]++ % it->second.size()];
    }
    return out;
}

extern "C" fsw_status fsw_policy_stripe_deal(uint32_t n_units, const int32_t* unit_node, uint32_t n_src,
                                             const int32_t* src_node, uint32_t* out) {
    if ((n_units && (!unit_node || !out)) || n_src == 0 || !src_node)
        return FSW_EINVAL;
    const std::vector<uint32_t> r = fsw::stripe_deal(std::vector<int>(unit_node, unit_node + n_units),
                                                     std::vector<int>(src_node, src_node + n_src));
    std::copy(r.begin(), r.end(), out);
    return FSW_OK;
}

extern "C" fsw_status fsw_policy_heavy(double swap_ms, double resident_ms, double deadline_ms, double queue_budget_ms,
                                       double theta, int32_t* heavy) {
    if (!heavy || !(swap_ms >= 0.0) || !(resident_ms >= 0.0) || !(theta > 0.0) || !(queue_budget_ms >= 0.0))
        return FSW_EINVAL;
    *heavy = heavy_by_slo(swap_ms, resident_ms, deadline_ms, queue_budget_ms, theta) ? 1 : 0;
    return FSW_OK;
}

extern "C" fsw_status fsw_policy_eviction_order(uint32_t n, const uint8_t* heavy, const uint32_t* copies,
                                                const uint64_t* last_use, const uint8_t* in_use, uint32_t* order,
                                                uint32_t* n_order) {
    if (!n_order || (n && (!heavy || !copies || !last_use || !in_use || !order))) return FSW_EINVAL;
    const std::vector<uint32_t> o = eviction_order(std::vector<uint8_t>(heavy, heavy + n), std::vector<uint32_t>(copies, copies + n),
                                                   std::vector<uint64_t>(last_use, last_use + n),
                                                   std::vector<uint8_t>(in_use, in_use + n));
    std::copy(o.begin(), o.end(), order);
    *n_order = (uint32_t)o.size();
    return FSW_OK;
}

// ==========================================================================================
// request scheduler
// ==========================================================================================
namespace {

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

struct Req {
    uint32_t fid;
    uint32_t model;  // copied at submit: workers never touch s->funcs outside the lock
    uint64_t ticket;
    const void* in;
    uint64_t in_bytes;
    void* out;
    uint64_t out_cap;
    double t_submit, t_start = 0, t_end = 0;
    bool done = false;
    fsw_request_stats st{};
};

struct Func {
    uint32_t model;
    double deadline_ms, p;
    uint64_t n = 0, m = 0;           // completed requests, of which within the deadline
    uint64_t n_period = 0, m_period = 0;
    double lat_sum = 0;
    std::deque<Req*> q;
};

}  // namespace

struct fsw_sched {
    fsw_ctx* ctx;
    fsw_sched_config cfg;
    std::mutex mu;
    std::condition_variable cv_disp, cv_work, cv_done;
    std::vector<Func> funcs;
    std::map<uint64_t, Req*> reqs;
    std::deque<Req*> work;            // dispatched, waiting for a worker
    uint64_t next_ticket = 1;
    uint32_t inflight = 0, max_inflight = 1;
    double alpha, last_ratio = -1.0, period_start = 0;
    bool stop = false;
    uint64_t completed = 0, met = 0, kinds[4] = {0, 0, 0, 0};
    std::thread dispatcher;
    std::vector<std::thread> workers;
};

static double norm_rrc(const Func& f) {
    const double avg = f.n ? f.lat_sum / (double)f.n : 1.0;  // SPEC normalized_rrc: RRC x mean latency
    return rrc(f.n, f.m, f.p) * avg;
}

// Next request: high-priority functions first, in reverse RRC order, then the
// low-priority ones in RRC order; FIFO within a function; ties by function id.
static Req* pick_next(fsw_sched* s) {
    std::vector<double> r(s->funcs.size());
    for (size_t i = 0; i < r.size(); ++i) r[i] = norm_rrc(s->funcs[i]);
    const std::vector<uint8_t> high = partition_high(r, s->alpha);
    int best = -1;
    for (int i = 0; i < (int)s->funcs.size(); ++i) {
        if (s->funcs[i].q.empty()) continue;
        if (best < 0) {
            best = i;
            continue;
        }
        const bool hi = high[i], hb = high[best];
        if (hi != hb) {
            if (hi) best = i;
        } else if (hi ? r[i] > r[best] : r[i] < r[best]) {
            best = i;
        }
    }
    if (best < 0) return nullptr;
    Req* q = s->funcs[best].q.front();
    s->funcs[best].q.pop_front();
    return q;
}

static void period_tick(fsw_sched* s, double t) {
    if (t - s->period_start < s->cfg.period_ms) return;
    uint32_t active = 0, ok = 0;
    for (Func& f : s->funcs) {
        if (f.n_period) {
            ++active;
            ok += (double)f.m_period >= f.p * (double)f.n_period;
        }
        f.n_period = f.m_period = 0;
    }
    if (active) {
        const double ratio = (double)ok / active;
        if (s->last_ratio >= 0) s->alpha = alpha_config(s->alpha, s->last_ratio, ratio, s->cfg.scalar, s->cfg.threshold);
        s->last_ratio = ratio;
    }
    s->period_start = t;
}

static void dispatcher_main(fsw_sched* s) {
    std::unique_lock<std::mutex> lk(s->mu);
    for (;;) {
        bool pending = false;
        for (const Func& f : s->funcs) pending |= !f.q.empty();
        if (s->stop && !pending) break;
        if (!pending || s->inflight >= s->max_inflight) {
            s->cv_disp.wait_for(lk, std::chrono::milliseconds((int64_t)std::max(1.0, s->cfg.period_ms)));
            period_tick(s, now_ms());
            continue;
        }
        period_tick(s, now_ms());
        Req* r = pick_next(s);
        if (!r) continue;
        s->inflight++;
        s->work.push_back(r);
        s->cv_work.notify_one();
    }
    s->cv_work.notify_all();
}

static void worker_main(fsw_sched* s) {
    for (;;) {
        Req* r = nullptr;
        {
            std::unique_lock<std::mutex> lk(s->mu);
            s->cv_work.wait(lk, [&] { return !s->work.empty() || (s->stop && s->inflight == 0); });
            if (s->work.empty()) return;
            r = s->work.front();
            s->work.pop_front();
            r->t_start = now_ms();
        }
        fsw_invoke_stats st{};
        const fsw_status rc = fsw_invoke(s->ctx, r->model, r->in, r->in_bytes, r->out, r->out_cap, &st);
        const double t_end = now_ms();
        std::lock_guard<std::mutex> lk(s->mu);
        Func& f = s->funcs[r->fid];
        r->t_end = t_end;
        r->st.status = rc;
        r->st.queue_ms = r->t_start - r->t_submit;
        r->st.total_ms = t_end - r->t_submit;
        r->st.gpu = st.gpu;
        r->st.swap_kind = st.swap_kind;
        r->st.device_ms = st.device_ms;
        // a request counts towards n at completion; it is compliant if it finished by its deadline
        r->st.met_deadline = rc == FSW_OK && r->st.total_ms <= f.deadline_ms;
        f.n++;
        f.n_period++;
        f.lat_sum += r->st.total_ms;
        if (r->st.met_deadline) {
            f.m++;
            f.m_period++;
            s->met++;
        }
        s->completed++;
        if (rc == FSW_OK && st.swap_kind < 4) s->kinds[st.swap_kind]++;
        r->done = true;
        s->inflight--;
        s->cv_disp.notify_all();
        s->cv_done.notify_all();
        if (s->stop && s->inflight == 0) s->cv_work.notify_all();
    }
}

extern "C" fsw_status fsw_sched_create(fsw_ctx* ctx, const fsw_sched_config* cfg, fsw_sched** out) {
    if (!ctx || !out) return FSW_EINVAL;
    uint32_t n_gpus = 0;
    if (fsw_n_gpus(ctx, &n_gpus) != FSW_OK || n_gpus == 0) return FSW_ECUDA;
    auto* s = new fsw_sched();
    s->ctx = ctx;
    s->cfg = cfg ? *cfg : fsw_sched_config{};
    if (s->cfg.alpha0 <= 0 || s->cfg.alpha0 > 1) s->cfg.alpha0 = 0.5;
    if (s->cfg.scalar <= 1) s->cfg.scalar = 2.0;          // Appendix B defaults
    if (s->cfg.threshold <= 0) s->cfg.threshold = 0.04;
    if (s->cfg.period_ms <= 0) s->cfg.period_ms = 10000;
    s->max_inflight = s->cfg.max_inflight ? s->cfg.max_inflight : n_gpus;
    s->alpha = s->cfg.alpha0;
    s->period_start = now_ms();
    s->dispatcher = std::thread(dispatcher_main, s);
    for (uint32_t i = 0; i < s->max_inflight; ++i) s->workers.emplace_back(worker_main, s);
    *out = s;
    return FSW_OK;
}

extern "C" void fsw_sched_destroy(fsw_sched* s) {
    if (!s) return;
    {
        std::lock_guard<std::mutex> lk(s->mu);
        s->stop = true;
    }
    s->cv_disp.notify_all();
    s->dispatcher.join();
    s->cv_work.notify_all();
    for (auto& t : s->workers) t.join();
    for (auto& kv : s->reqs) delete kv.second;
    delete s;
}

extern "C" fsw_status fsw_function_register(fsw_sched* s, uint32_t model_id, double deadline_ms, double p, uint32_t* fid) {
    if (!s || !fid || !(deadline_ms > 0) || !(p > 0 && p < 1)) return FSW_EINVAL;
    fsw_model_info mi;
    if (fsw_model_info_get(s->ctx, model_id, &mi) != FSW_OK) return FSW_ENOTFOUND;
    // the model's class is judged against its tightest deadline
    if (fsw_model_set_slo(s->ctx, model_id, deadline_ms) != FSW_OK) return FSW_ENOTFOUND;
    std::lock_guard<std::mutex> lk(s->mu);
    Func f;
    f.model = model_id;
    f.deadline_ms = deadline_ms;
    f.p = p;
    s->funcs.push_back(f);
    *fid = (uint32_t)s->funcs.size() - 1;
    return FSW_OK;
}

extern "C" fsw_status fsw_submit(fsw_sched* s, uint32_t fid, const void* input, uint64_t in_bytes, void* output,
                                 uint64_t out_cap, uint64_t* ticket) {
    if (!s || !ticket || !input || !output) return FSW_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    if (fid >= s->funcs.size()) return FSW_ENOTFOUND;
    if (s->stop) return FSW_ESTATE;
    Req* r = new Req{fid, s->funcs[fid].model, s->next_ticket++, input, in_bytes, output, out_cap, now_ms()};
    s->reqs[r->ticket] = r;
    s->funcs[fid].q.push_back(r);
    *ticket = r->ticket;
    s->cv_disp.notify_all();
    return FSW_OK;
}

extern "C" fsw_status fsw_wait(fsw_sched* s, uint64_t ticket, fsw_request_stats* out) {
    if (!s) return FSW_EINVAL;
    std::unique_lock<std::mutex> lk(s->mu);
    auto it = s->reqs.find(ticket);
    if (it == s->reqs.end()) return FSW_ENOTFOUND;
    Req* r = it->second;
    s->cv_done.wait(lk, [&] { return r->done; });
    if (out) *out = r->st;
    const fsw_status rc = r->st.status;
    s->reqs.erase(it);
    delete r;
    return rc;
}

extern "C" fsw_status fsw_function_stats_get(fsw_sched* s, uint32_t fid, fsw_function_stats* out) {
    if (!s || !out) return FSW_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    if (fid >= s->funcs.size()) return FSW_ENOTFOUND;
    std::vector<double> r(s->funcs.size());
    for (size_t i = 0; i < r.size(); ++i) r[i] = norm_rrc(s->funcs[i]);
    const Func& f = s->funcs[fid];
    out->n = f.n;
    out->m = f.m;
    out->rrc = rrc(f.n, f.m, f.p);
    out->rrc_normalized = r[fid];
    out->avg_latency_ms = f.n ? f.lat_sum / (double)f.n : 0.0;
    out->high = partition_high(r, s->alpha)[fid];
    out->queued = (uint32_t)f.q.size();
    return FSW_OK;
}

extern "C" fsw_status fsw_sched_stats_get(fsw_sched* s, fsw_sched_stats* out) {
    if (!s || !out) return FSW_EINVAL;
    std::lock_guard<std::mutex> lk(s->mu);
    memset(out, 0, sizeof *out);
    out->alpha = s->alpha;
    out->n_functions = (uint32_t)s->funcs.size();
    std::vector<double> r(s->funcs.size());
    uint32_t active = 0, ok = 0;
    for (size_t i = 0; i < r.size(); ++i) {
        const Func& f = s->funcs[i];
        r[i] = norm_rrc(f);
        if (f.n) {
            ++active;
            ok += (double)f.m >= f.p * (double)f.n;
        }
    }
    for (uint8_t h : partition_high(r, s->alpha)) out->n_high += h;
    out->completed = s->completed;
    out->met_deadline = s->met;
    out->slo_compliant_functions = ok;
    out->active_functions = active;
    out->n_resident = s->kinds[FSW_SWAP_RESIDENT];
    out->n_host_swaps = s->kinds[FSW_SWAP_HOST];
    out->n_peer_swaps = s->kinds[FSW_SWAP_PEER];
    out->n_striped_swaps = s->kinds[FSW_SWAP_STRIPED];
    return FSW_OK;
}
