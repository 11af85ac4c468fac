// control.cpp — host control plane of the Sync-Switch path: Table I remap, seeded arrival schedule, straggler
// detector and greedy policy. Host-only C++ (no CUDA); exported through include/syncswitch.h.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <new>
#include <vector>

#include "plan.h"
#include "syncswitch.h"

namespace ss {

int32_t Layout::first_hosted(int32_t r) const {
  int32_t j = 0;
  while (j < n && host(j) < r) ++j;
  return j;
}

int32_t Layout::n_hosted(int32_t r) const {
  int32_t c = 0;
  for (int32_t j = 0; j < n; ++j) c += host(j) == r;
  return c;
}

Layout make_layout(int64_t P, int32_t S, int32_t n, int32_t rank, int32_t world) {
  Layout L;
  L.rank = rank;
  L.world = world;
  L.n = n;
  L.S = S;
  L.P = P;
  L.pad = (((P + S - 1) / S) + 31) / 32 * 32;
  L.P_pad = L.pad * S;
  L.reg_len = L.P_pad / world;
  L.real_lo.resize(world);
  L.real_hi.resize(world);
  for (int32_t r = 0; r < world; ++r) {
    L.real_lo[r] = std::min<int64_t>((int64_t)r * L.reg_len, P);
    L.real_hi[r] = std::min<int64_t>((int64_t)(r + 1) * L.reg_len, P);
  }
  return L;
}

void plan_window(const Layout &L, const int32_t *kind, const int32_t *worker, const uint8_t *data, int32_t n_ev,
                 std::vector<RouteOp> &out) {
  const int32_t me = L.rank;
  for (int32_t k = 0; k < n_ev; ++k) {  // phase 0: every push's slices to their owners
    if (kind[k] != 0) continue;
    const int32_t h = L.host(worker[k]);
    if (h == me) {
      for (int32_t r = 0; r < L.world; ++r)
        if (r != me && L.count(r) > 0) out.push_back({0, 0, r, k, L.real_lo[r], L.count(r)});
    } else if (L.count(me) > 0) {
      out.push_back({0, 1, h, k, L.real_lo[me], L.count(me)});
    }
  }
  for (int32_t k = 0; k < n_ev; ++k) {  // phase 1: every pull's snapshot slices to the puller
    if (kind[k] != 1 || !data[k]) continue;
    const int32_t h = L.host(worker[k]);
    if (h == me) {
      for (int32_t r = 0; r < L.world; ++r)
        if (r != me && L.count(r) > 0) out.push_back({1, 1, r, k, L.real_lo[r], L.count(r)});
    } else if (L.count(me) > 0) {
      out.push_back({1, 0, h, k, L.real_lo[me], L.count(me)});
    }
  }
}

bool window_cut(const int32_t *kind, const int32_t *worker, int32_t n_in_window, int32_t new_kind, int32_t new_worker,
                int32_t max_window, bool fused) {
  if (n_in_window >= max_window) return true;
  if (fused && new_kind == 1)
    for (int32_t k = 0; k < n_in_window; ++k)
      if (kind[k] == 1 && worker[k] == new_worker) return true;
  return false;
}

}  // namespace ss

namespace {

uint64_t mix64(uint64_t x) {  // splitmix64 finaliser with the golden-gamma increment
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

extern "C" {

// Table I with the piecewise boundary rule (DESIGN reading C11).
ss_status ss_table1(int64_t W, int64_t B, int64_t N, int64_t s_num, int64_t s_den, const int64_t *Wb, int32_t nb,
                    int64_t *bsp_steps, int64_t *asp_steps, int64_t *bounds_out) {
  if (W <= 0 || B <= 0 || N <= 0 || s_den <= 0 || s_num < 0 || s_num > s_den || nb < 0 || !bsp_steps ||
      !asp_steps || (nb > 0 && (!Wb || !bounds_out)))
    return SS_E_INVAL;
  const __int128 ws_num = (__int128)W * s_num;
  if (ws_num % s_den) return SS_E_INVAL;
  const int64_t bsp_samples = (int64_t)(ws_num / s_den);  // W*s samples trained with BSP
  const int64_t global_batch = B * N;                     // BSP batch nB
  if (bsp_samples % global_batch || W % B) return SS_E_INVAL;
  *bsp_steps = bsp_samples / global_batch;
  *asp_steps = (W - bsp_samples) / B;
  for (int32_t i = 0; i < nb; ++i) {
    const int64_t wi = Wb[i];
    if (wi <= bsp_samples) {  // the boundary falls inside the BSP phase: count it in BSP steps
      if (wi % global_batch) return SS_E_INVAL;
      bounds_out[i] = wi / global_batch;
    } else {                   // after the switch: BSP steps + ASP steps of the remaining samples
      if ((wi - bsp_samples) % B) return SS_E_INVAL;
      bounds_out[i] = *bsp_steps + (wi - bsp_samples) / B;
    }
  }
  return SS_OK;
}

// Seeded integer-tick arrival schedule (DESIGN reading C7). A per-worker "next push" clock; each step emits the
// earliest (tick, worker) push followed by that worker's pull.
ss_status ss_schedule(int32_t n, const int64_t *period, int64_t jitter, uint64_t seed, int32_t slow_worker,
                      int64_t slow_factor, int64_t slow_t0, int64_t slow_t1, int64_t n_push, int32_t *kind,
                      int32_t *worker, int64_t *tick, int64_t *n_out) {
  if (n < 1 || n > 256 || !period || jitter < 0 || n_push < 0 || !kind || !worker || !tick || !n_out ||
      slow_factor < 1)
    return SS_E_INVAL;
  for (int32_t j = 0; j < n; ++j)
    if (period[j] <= jitter) return SS_E_INVAL;  // every gap T + d must stay positive
  auto gap = [&](int32_t j, int64_t at, int64_t k) -> int64_t {
    int64_t T = period[j];
    if (j == slow_worker && at >= slow_t0 && at < slow_t1) T *= slow_factor;
    int64_t d = 0;
    if (jitter > 0) {
      const uint64_t h = mix64(seed ^ ((uint64_t)(uint32_t)j << 32) ^ (uint64_t)k);
      d = (int64_t)(h % (uint64_t)(2 * jitter + 1)) - jitter;
    }
    return T + d;
  };
  std::vector<int64_t> next(n), pushes(n, 0);
  int64_t e = 0;
  for (int32_t j = 0; j < n; ++j) {
    kind[e] = 1; worker[e] = j; tick[e] = 0; ++e;
    next[j] = gap(j, 0, 1);
  }
  for (int64_t p = 0; p < n_push; ++p) {
    int32_t b = 0;
    for (int32_t j = 1; j < n; ++j)
      if (next[j] < next[b]) b = j;
    const int64_t t = next[b];
    kind[e] = 0; worker[e] = b; tick[e] = t; ++e;
    kind[e] = 1; worker[e] = b; tick[e] = t; ++e;
    pushes[b] += 1;
    next[b] = t + gap(b, t, pushes[b] + 1);
  }
  *n_out = e;
  return SS_OK;
}

struct ss_detector {
  int32_t n, K;
  std::vector<int32_t> run;
  int32_t clean = 0;
};

ss_status ss_detector_new(ss_detector **out, int32_t n, int32_t K) {
  if (!out || n < 1 || K < 1) return SS_E_INVAL;
  ss_detector *d = new (std::nothrow) ss_detector;
  if (!d) return SS_E_INVAL;
  d->n = n;
  d->K = K;
  d->run.assign(n, 0);
  *out = d;
  return SS_OK;
}

// S_k over the window; flagged when S_k < S - sigma (population sigma, reading C14); a straggler after K
// consecutive flagged windows. Cluster clean after K windows without any flag (reading C15). With a mask, only the
// masked-in workers are measured (elastic policy): the others are neither in S, sigma nor flagged.
ss_status ss_detector_window_masked(ss_detector *d, const double *samples, const double *busy, const uint8_t *mask,
                                    int32_t *straggler, int32_t *clean_out) {
  if (!d || !samples || !busy || !straggler) return SS_E_INVAL;
  std::vector<double> s(d->n);
  double mean = 0.0;
  int32_t m = 0;
  for (int32_t k = 0; k < d->n; ++k) {
    s[k] = busy[k] > 0.0 ? samples[k] / busy[k] : 0.0;
    if (!mask || mask[k]) {
      mean += s[k];
      ++m;
    }
  }
  mean = m > 0 ? mean / m : 0.0;
  double ss = 0.0;
  for (int32_t k = 0; k < d->n; ++k)
    if (!mask || mask[k]) ss += (s[k] - mean) * (s[k] - mean);
  const double thr = mean - std::sqrt(m > 0 ? ss / m : 0.0);
  bool any = false;
  for (int32_t k = 0; k < d->n; ++k) {
    const bool in = !mask || mask[k];
    const bool f = in && s[k] < thr;
    d->run[k] = f ? d->run[k] + 1 : 0;
    straggler[k] = d->run[k] >= d->K;
    any = any || f;
  }
  d->clean = any ? 0 : d->clean + 1;
  if (clean_out) *clean_out = d->clean >= d->K;
  return SS_OK;
}

ss_status ss_detector_window(ss_detector *d, const double *samples, const double *busy, int32_t *straggler,
                             int32_t *clean_out) {
  return ss_detector_window_masked(d, samples, busy, nullptr, straggler, clean_out);
}

void ss_detector_free(ss_detector *d) { delete d; }

// Routing plan of a whole ASP event sequence as seen by `rank` (window cuts + per-window ops), for CPU tests of the
// multi-GPU host logic. Window k of the sequence is reported in ops[i].window; event indices are window-relative.
ss_status ss_route_plan(int32_t rank, int32_t world, int32_t n_workers, int32_t n_shards, int64_t n_params,
                        int32_t max_window, int32_t fused, const int32_t *kind, const int32_t *worker, int64_t n_ev,
                        ss_route_op *ops, int64_t cap, int64_t *n_ops, int32_t *n_windows) {
  if (world < 1 || rank < 0 || rank >= world || n_workers < 1 || n_shards < 1 || n_shards % world || n_params < 1 ||
      max_window < 1 || max_window > 64 || n_ev < 0 || (n_ev > 0 && (!kind || !worker)) || !n_ops || cap < 0 ||
      (cap > 0 && !ops))
    return SS_E_INVAL;
  const ss::Layout L = ss::make_layout(n_params, n_shards, n_workers, rank, world);
  std::vector<int32_t> wk, ww;
  std::vector<uint8_t> wd;
  std::vector<ss::RouteOp> plan;
  int64_t total = 0;
  int32_t win_id = 0;
  auto emit = [&]() {
    if (wk.empty()) return;
    plan.clear();
    ss::plan_window(L, wk.data(), ww.data(), wd.data(), (int32_t)wk.size(), plan);
    for (const ss::RouteOp &o : plan) {
      if (total < cap) ops[total] = ss_route_op{win_id, o.phase, o.op, o.peer, o.event, o.offset, o.count};
      ++total;
    }
    ++win_id;
    wk.clear();
    ww.clear();
    wd.clear();
  };
  for (int64_t i = 0; i < n_ev; ++i) {
    if (ss::window_cut(wk.data(), ww.data(), (int32_t)wk.size(), kind[i], worker[i], max_window, fused != 0)) emit();
    wk.push_back(kind[i]);
    ww.push_back(worker[i]);
    wd.push_back(1);
    if ((int32_t)wk.size() >= max_window) emit();
  }
  emit();
  *n_ops = total;
  if (n_windows) *n_windows = win_id;
  return SS_OK;
}

// Dynamic switching rule: satisfied when |Delta| < c*sigma (|Delta| = 0 counts as satisfied);
// fires after T consecutive satisfied steps.
int32_t ss_criterion_observe(int32_t *run, float norm_delta, float sigma, float c, int32_t T) {
  if (!run || T < 1) return 0;
  const bool ok = norm_delta == 0.0f || (double)norm_delta < (double)c * (double)sigma;
  *run = ok ? *run + 1 : 0;
  return *run >= T;
}

// Greedy policy: "simply switches to ASP ... when a straggler is detected; once the cluster is free of any
// stragglers and the aggregate BSP training has not been satisfied, it will switch back to training with BSP".
int32_t ss_greedy_decision(int32_t protocol, int32_t any_straggler, int32_t cluster_clean, int64_t bsp_done,
                           int64_t bsp_quota) {
  if (protocol == SS_BSP && any_straggler && bsp_done < bsp_quota) return SS_ASP;
  if (protocol == SS_ASP && cluster_clean && bsp_done < bsp_quota) return SS_BSP;
  return -1;
}

}  // extern "C"
