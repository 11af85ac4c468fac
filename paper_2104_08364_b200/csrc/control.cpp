// control.cpp — host control plane of the Sync-Switch path: Table I remap, seeded arrival schedule, straggler
// detector and greedy policy. Host-only C++ (no CUDA); exported through include/syncswitch.h.
#include <cmath>
#include <cstdint>
#include <new>
#include <vector>

#include "syncswitch.h"

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
// consecutive flagged windows. Cluster clean after K windows without any flag (reading C15).
ss_status ss_detector_window(ss_detector *d, const double *samples, const double *busy, int32_t *straggler,
                             int32_t *clean_out) {
  if (!d || !samples || !busy || !straggler) return SS_E_INVAL;
  std::vector<double> s(d->n);
  double mean = 0.0;
  for (int32_t k = 0; k < d->n; ++k) {
    s[k] = busy[k] > 0.0 ? samples[k] / busy[k] : 0.0;
    mean += s[k];
  }
  mean /= d->n;
  double ss = 0.0;
  for (int32_t k = 0; k < d->n; ++k) ss += (s[k] - mean) * (s[k] - mean);
  const double thr = mean - std::sqrt(ss / d->n);
  bool any = false;
  for (int32_t k = 0; k < d->n; ++k) {
    const bool f = s[k] < thr;
    d->run[k] = f ? d->run[k] + 1 : 0;
    straggler[k] = d->run[k] >= d->K;
    any = any || f;
  }
  d->clean = any ? 0 : d->clean + 1;
  if (clean_out) *clean_out = d->clean >= d->K;
  return SS_OK;
}

void ss_detector_free(ss_detector *d) { delete d; }

// Greedy policy: "simply switches to ASP ... when a straggler is detected; once the cluster is free of any
// stragglers and the aggregate BSP training has not been satisfied, it will switch back to training with BSP".
int32_t ss_greedy_decision(int32_t protocol, int32_t any_straggler, int32_t cluster_clean, int64_t bsp_done,
                           int64_t bsp_quota) {
  if (protocol == SS_BSP && any_straggler && bsp_done < bsp_quota) return SS_ASP;
  if (protocol == SS_ASP && cluster_clean && bsp_done < bsp_quota) return SS_BSP;
  return -1;
}

}  // extern "C"
