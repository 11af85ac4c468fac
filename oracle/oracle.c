/*
 * oracle.c — plain, slow, single-threaded CPU oracle of the Sync-Switch synchronization path.
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs; never by the product path. Shares nothing with paper_2104_08364_b200/.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -std=c11 -shared -fPIC oracle.c -lm -o liboracle.so
 * (-ffp-contract=off: every fused multiply-add is the explicit fmaf()/fma() the text below writes; nothing else
 * is contracted, so float arithmetic is exactly what is written, in the order written).
 *
 * Parity status per function:
 *   shard layout, lr, Table I, state machine, synth grad, schedule, detector: pinned (tests/test_oracle_*.py).
 *   softmax toy model: pinned by closed forms (ln C at W=0) and central finite differences.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------------------------
 * Shard layout. P:15 "one needs to divide the model parameters into different shards, each shard managed by one
 * PS instance"; the method is a TODO in the paper, so SURVEY §8 fixes it: equal contiguous shards padded
 * to 32 floats (128 B), owner(s) = floor(s*G/S), host(j) = floor(j*G/n). */
int64_t orc_shard_pad(int64_t P, int32_t S) {
  int64_t per = (P + S - 1) / S;          /* ceil(P/S) */
  return ((per + 31) / 32) * 32;          /* round up to 32 floats */
}

void orc_shard_offsets(int64_t P, int32_t S, int64_t *off) {
  int64_t pad = orc_shard_pad(P, S);
  for (int32_t s = 0; s <= S; s++) {
    int64_t o = (int64_t)s * pad;
    off[s] = o < P ? o : P;
  }
}

int32_t orc_shard_owner(int32_t s, int32_t S, int32_t G) { return (int32_t)(((int64_t)s * G) / S); }
int32_t orc_worker_host(int32_t j, int32_t n, int32_t G) { return (int32_t)(((int64_t)j * G) / n); }

/* ------------------------------------------------------------------------------------------------------------
 * Learning rate. P:1600: "learning rate to be 0.1 and decays ... at 32K and 48K steps with scaling factors of 0.1
 * and 0.01"; factors multiply the base rate, not each other ("not cumulative"); right-continuous. */
double orc_lr_factor(int64_t version, const int64_t *bounds, const float *factors, int32_t nb) {
  double f = 1.0;
  for (int32_t i = 0; i < nb; i++)
    if (bounds[i] <= version) f = (double)factors[i];
  return f;
}

/* P:1473 "eta_BSP = n*eta" (linear scaling rule); "eta_ASP = eta/sqrt(n)" (reading C3: rule 0 = 1/sqrt(n),
 * rule 1 = 1/n, rule 2 = unscaled). Computed in double, rounded to float once. */
float orc_lr(float eta, double factor, int32_t proto, int32_t n, int32_t asp_rule) {
  double scale;
  if (proto == ORC_BSP) scale = (double)n;
  else if (asp_rule == 0) scale = 1.0 / sqrt((double)n);
  else if (asp_rule == 1) scale = 1.0 / (double)n;
  else scale = 1.0;
  return (float)((double)eta * factor * scale);
}

/* Table I: BSP steps = W*s/(B*N); ASP steps = W/B - W*s/B; a decay boundary W_i (in samples) moves to
 * W_i/B - W*s/B + W*s/(B*N) when it lies after the BSP share, else to W_i/(B*N) (reading C11: the draft's single
 * formula gives negative boundaries for rows 75-25 and 100-0; the piecewise rule reproduces all 11 rows). */
int32_t orc_table1(int64_t W, int64_t B, int64_t N, int64_t s_num, int64_t s_den, const int64_t *Wb, int32_t nb,
                   int64_t *bsp_steps, int64_t *asp_steps, int64_t *bounds_out) {
  if (W <= 0 || B <= 0 || N <= 0 || s_den <= 0 || s_num < 0 || s_num > s_den) return -1;
  /* Ws = W*s samples processed under BSP; must be integral, as must the step counts. */
  if ((W * s_num) % s_den != 0) return -1;
  int64_t Ws = W * s_num / s_den;
  if (Ws % (B * N) != 0 || W % B != 0 || Ws % B != 0) return -1;
  *bsp_steps = Ws / (B * N);
  *asp_steps = W / B - Ws / B;
  for (int32_t i = 0; i < nb; i++) {
    if (Wb[i] % B != 0) return -1;
    if (Wb[i] <= Ws) {
      if (Wb[i] % (B * N) != 0) return -1;
      bounds_out[i] = Wb[i] / (B * N);
    } else {
      bounds_out[i] = Wb[i] / B - Ws / B + Ws / (B * N);
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------------------------
 * The state machine, instantiated for float (parity) and double (identities). */
#define REAL float
#define ORC_T orc_f
#define ORC_FN(x) orcf##x
#define ORC_FMA fmaf
#include "oracle_state.inc"
#undef REAL
#undef ORC_T
#undef ORC_FN
#undef ORC_FMA

#define REAL double
#define ORC_T orc_d
#define ORC_FN(x) orcd##x
#define ORC_FMA fma
#include "oracle_state.inc"
#undef REAL
#undef ORC_T
#undef ORC_FN
#undef ORC_FMA

/* ------------------------------------------------------------------------------------------------------------
 * Synthetic inputs, written from their stated formulas. splitmix64 = Steele/Lea/Flood's finaliser
 * with the golden-gamma increment. */
uint64_t orc_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void orc_synth_grad(uint64_t seed, int32_t j, int64_t k, int64_t i0, int64_t count, float *out) {
  for (int64_t t = 0; t < count; t++) {
    uint64_t i = (uint64_t)(i0 + t);
    uint64_t key = ((uint64_t)(uint32_t)j << 56) ^ ((uint64_t)k << 30) ^ i;
    uint64_t h = orc_splitmix64(seed ^ key);
    double u = (double)(h >> 40) * (1.0 / 16777216.0);  /* 24-bit integer * 2^-24, exact */
    out[t] = (float)((u - 0.5) * (1.0 / 64.0));         /* exact in float: 24 significant bits at most */
  }
}

/* Arrival schedule (reading C7). Plain event simulation: keep each worker's next push tick; repeatedly take the
 * smallest (tick, worker); emit push then the same worker's pull. */
int64_t orc_schedule(int32_t n, const int64_t *period, int64_t jitter, uint64_t seed, int32_t slow_worker,
                     int64_t slow_factor, int64_t slow_t0, int64_t slow_t1, int64_t n_push, int32_t *ev_kind,
                     int32_t *ev_worker, int64_t *ev_tick) {
  int64_t *next = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  int64_t *count = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  int64_t e = 0;
  for (int32_t j = 0; j < n; j++) {          /* every worker pulls at t = 0 */
    ev_kind[e] = 1; ev_worker[e] = j; ev_tick[e] = 0; e++;
  }
  for (int32_t j = 0; j < n; j++) {
    int64_t prev = 0, k = 1;
    int64_t T = period[j];
    if (j == slow_worker && prev >= slow_t0 && prev < slow_t1) T *= slow_factor;
    int64_t d = 0;
    if (jitter > 0)
      d = (int64_t)(orc_splitmix64(seed ^ ((uint64_t)(uint32_t)j << 32) ^ (uint64_t)k) % (uint64_t)(2 * jitter + 1)) -
          jitter;
    next[j] = prev + T + d;
  }
  for (int64_t p = 0; p < n_push; p++) {
    int32_t best = 0;
    for (int32_t j = 1; j < n; j++)
      if (next[j] < next[best]) best = j;      /* ties broken by the lower worker id */
    int64_t t = next[best];
    ev_kind[e] = 0; ev_worker[e] = best; ev_tick[e] = t; e++;
    ev_kind[e] = 1; ev_worker[e] = best; ev_tick[e] = t; e++;
    count[best] += 1;
    int64_t k = count[best] + 1;
    int64_t T = period[best];
    if (best == slow_worker && t >= slow_t0 && t < slow_t1) T *= slow_factor;
    int64_t d = 0;
    if (jitter > 0)
      d = (int64_t)(orc_splitmix64(seed ^ ((uint64_t)(uint32_t)best << 32) ^ (uint64_t)k) %
                    (uint64_t)(2 * jitter + 1)) -
          jitter;
    next[best] = t + T + d;
  }
  free(next);
  free(count);
  return e;
}

/* ------------------------------------------------------------------------------------------------------------
 * Toy model: softmax regression (SURVEY config 1; stands in for the worker's forward/backward). fp64. */
double orc_softmax_loss_grad(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const double *W,
                             double *grad) {
  double *z = (double *)malloc((size_t)C * sizeof(double));
  double loss = 0.0;
  for (int64_t i = 0; i < (int64_t)d * C; i++) grad[i] = 0.0;
  for (int32_t b = 0; b < B; b++) {
    const float *x = X + (int64_t)b * d;
    for (int32_t c = 0; c < C; c++) {            /* logits z = x W */
      double acc = 0.0;
      for (int32_t i = 0; i < d; i++) acc += (double)x[i] * W[(int64_t)i * C + c];
      z[c] = acc;
    }
    double m = z[0];
    for (int32_t c = 1; c < C; c++) if (z[c] > m) m = z[c];
    double den = 0.0;
    for (int32_t c = 0; c < C; c++) den += exp(z[c] - m);
    loss += -((z[y[b]] - m) - log(den));         /* -log p_{b,y_b} */
    for (int32_t c = 0; c < C; c++) {
      double p = exp(z[c] - m) / den;
      double r = (p - (c == y[b] ? 1.0 : 0.0)) / (double)B;
      for (int32_t i = 0; i < d; i++) grad[(int64_t)i * C + c] += (double)x[i] * r;   /* X^T (p - Y) / B */
    }
  }
  free(z);
  return loss / (double)B;
}

/* ------------------------------------------------------------------------------------------------------------
 * Straggler detection ("a worker k is identified as a straggler if its training throughput over a sliding
 * window S_k is lower than the difference between the cluster average and standard deviation S - sigma, for a
 * number of consecutive detection windows"). sigma is the population standard deviation (reading C14). */
struct orc_detector {
  int32_t n, K;
  int32_t *run;        /* consecutive flagged windows per worker */
  int32_t clean_run;   /* consecutive windows with no worker flagged */
};

orc_detector *orc_detector_new(int32_t n, int32_t K) {
  if (n < 1 || K < 1) return NULL;
  orc_detector *dt = (orc_detector *)calloc(1, sizeof(orc_detector));
  dt->n = n; dt->K = K;
  dt->run = (int32_t *)calloc((size_t)n, sizeof(int32_t));
  return dt;
}

void orc_detector_free(orc_detector *dt) {
  if (!dt) return;
  free(dt->run);
  free(dt);
}

/* With a mask (elastic policy) only the workers still at the BSP barrier are measured: S and sigma are taken over
 * them, only they can be flagged, the others' consecutive counts restart. */
int32_t orc_detector_window_masked(orc_detector *dt, const double *samples, const double *busy, const uint8_t *mask,
                                   int32_t *straggler) {
  int32_t n = dt->n, counted = 0;
  double *Sk = (double *)malloc((size_t)n * sizeof(double));
  double mean = 0.0;
  for (int32_t k = 0; k < n; k++) {
    Sk[k] = busy[k] > 0.0 ? samples[k] / busy[k] : 0.0;
    if (mask == NULL || mask[k]) { mean += Sk[k]; counted++; }
  }
  if (counted > 0) mean /= (double)counted;
  double var = 0.0;
  for (int32_t k = 0; k < n; k++)
    if (mask == NULL || mask[k]) var += (Sk[k] - mean) * (Sk[k] - mean);
  double sigma = counted > 0 ? sqrt(var / (double)counted) : 0.0;
  int32_t any = 0;
  for (int32_t k = 0; k < n; k++) {
    int32_t flagged = (mask == NULL || mask[k]) && Sk[k] < mean - sigma;
    dt->run[k] = flagged ? dt->run[k] + 1 : 0;
    straggler[k] = dt->run[k] >= dt->K;
    any |= flagged;
  }
  dt->clean_run = any ? 0 : dt->clean_run + 1;
  free(Sk);
  return dt->clean_run >= dt->K;
}

int32_t orc_detector_window(orc_detector *dt, const double *samples, const double *busy, int32_t *straggler) {
  return orc_detector_window_masked(dt, samples, busy, NULL, straggler);
}

/* ------------------------------------------------------------------------------------------------------------
 * Online straggler scenario (config 4; DESIGN reading C23), written from its stated rules:
 *  - ticks are integers; worker j's k-th step lasts T_j(t) + d_{j,k} (T_j = period, x slow_factor for the slow worker
 *    while slow_t0 <= t < slow_t1; d as in the schedule), t = the time the step starts;
 *  - BSP superstep: all n workers compute from the same start time; the step ends at the slowest; each worker's busy
 *    time is its own duration; n*B samples;
 *  - ASP: each worker's next push happens when its step ends (earliest first, ties by lower id), then it pulls and
 *    starts its next step; B samples per push;
 *  - after every event, each detection window that ended at or before the current tick is evaluated in order with
 *    the samples / busy time of the steps completed inside it, then the greedy rule is applied;
 *  - the BSP share is the first W*q_num/q_den samples; meeting it switches to ASP for good;
 *  - a greedy switch back to BSP makes every worker's in-flight gradient arrive late (rejected, counted).
 * st == NULL: dry run (no data). Gradients: worker j's k-th gradient is orc_synth_grad(grad_seed, j, k, 0, P). */
int64_t orc_scenario_run(orc_f *st, int64_t P, int32_t n, int64_t B, int64_t W, int64_t q_num, int64_t q_den,
                         int64_t period, int64_t jitter, uint64_t sched_seed, uint64_t grad_seed, int32_t slow_worker,
                         int64_t slow_factor, int64_t slow_t0, int64_t slow_t1, int64_t D, int32_t K,
                         int32_t policy, int64_t *log5, int32_t cap, int64_t *res7) {
  int64_t quota = (W / q_den) * q_num + ((W % q_den) * q_num) / q_den;   /* floor(W * q_num / q_den) */
  int64_t *steps = (int64_t *)calloc((size_t)n, sizeof(int64_t));      /* gradients computed per worker */
  int64_t *base = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  int64_t *finish = (int64_t *)calloc((size_t)n, sizeof(int64_t));     /* ASP: when the running step ends */
  int64_t *length = (int64_t *)calloc((size_t)n, sizeof(int64_t));     /* ASP: its duration */
  double *win_samples = (double *)calloc((size_t)n, sizeof(double));
  double *win_busy = (double *)calloc((size_t)n, sizeof(double));
  int32_t *flag = (int32_t *)calloc((size_t)n, sizeof(int32_t));
  float **g = (float **)calloc((size_t)n, sizeof(float *));
  for (int32_t j = 0; j < n; j++) g[j] = st ? (float *)malloc((size_t)P * sizeof(float)) : NULL;
  int64_t *ver = (int64_t *)calloc((size_t)n, sizeof(int64_t));
  int32_t *ids = (int32_t *)calloc((size_t)n, sizeof(int32_t));
  uint8_t *active = (uint8_t *)malloc((size_t)n);       /* elastic: workers still at the BSP barrier */
  for (int32_t j = 0; j < n; j++) active[j] = 1;
  int32_t n_active = n;
  orc_detector *det = orc_detector_new(n, K);
  int64_t now = 0, processed = 0, bsp_samples = 0, version = 0, next_window = D;
  int64_t bsp_steps = 0, asp_pushes = 0, dropped = 0, windows = 0, nlog = 0;
  int32_t proto = ORC_BSP;

#define STEP_LEN(j, at)                                                                                       \
  ((((j) == slow_worker && (at) >= slow_t0 && (at) < slow_t1) ? period * slow_factor : period) +              \
   (jitter > 0 ? (int64_t)(orc_splitmix64(sched_seed ^ ((uint64_t)(uint32_t)(j) << 32) ^ (uint64_t)(steps[j] + 1)) % \
                           (uint64_t)(2 * jitter + 1)) - jitter                                                \
               : 0))
#define LOG_SWITCH(to, why)                      \
  do {                                           \
    if (st) orcf_switch(st, (to), 0);            \
    if (nlog < cap) {                            \
      log5[5 * nlog + 0] = now;                  \
      log5[5 * nlog + 1] = version;              \
      log5[5 * nlog + 2] = (to);                 \
      log5[5 * nlog + 3] = (why);                \
      log5[5 * nlog + 4] = n_active;             \
    }                                            \
    nlog++;                                      \
    proto = (to);                                \
  } while (0)
#define BEGIN_ASP()                                              \
  do {                                                           \
    for (int32_t q = 0; q < n; q++) {                            \
      if (st) orcf_pull(st, q, NULL, &base[q]);                  \
      else base[q] = version;                                    \
      length[q] = STEP_LEN(q, now);                              \
      finish[q] = now + length[q];                               \
    }                                                            \
  } while (0)

  while (processed < W) {
    if (proto == ORC_BSP) {
      int64_t slowest = 0;
      int32_t m = 0;
      for (int32_t j = 0; j < n; j++) {
        if (!active[j]) continue;                      /* removed workers receive no work */
        int64_t len = STEP_LEN(j, now);
        if (len > slowest) slowest = len;
        win_busy[j] += (double)len;
        win_samples[j] += (double)B;
        if (st) orc_synth_grad(grad_seed, j, steps[j], 0, P, g[m]);
        ids[m] = j;
        ver[m] = version;
        m++;
      }
      if (st) orcf_bsp_step(st, (const float *const *)g, ids, ver, m);
      for (int32_t j = 0; j < n; j++)
        if (active[j]) steps[j]++;
      version++;
      now += slowest;
      processed += (int64_t)m * B;
      bsp_samples += (int64_t)m * B;
      bsp_steps++;
      if (bsp_samples >= quota) {
        if (n_active < n) {                            /* restore the cluster size */
          for (int32_t j = 0; j < n; j++) { active[j] = 1; ids[j] = j; }
          n_active = n;
          if (st) orcf_set_members(st, ids, n);
        }
        LOG_SWITCH(ORC_ASP, 0);
        BEGIN_ASP();
      }
    } else {
      int32_t j = 0;
      for (int32_t q = 1; q < n; q++)
        if (finish[q] < finish[j]) j = q;
      now = finish[j];
      int64_t stale = 0;
      if (st) {
        orc_synth_grad(grad_seed, j, steps[j], 0, P, g[0]);
        orcf_asp_push(st, j, g[0], base[j], &stale);
      }
      steps[j]++;
      version++;
      if (st) orcf_pull(st, j, NULL, &base[j]);
      else base[j] = version;
      win_busy[j] += (double)length[j];
      win_samples[j] += (double)B;
      processed += B;
      asp_pushes++;
      length[j] = STEP_LEN(j, now);
      finish[j] = now + length[j];
    }
    while (next_window <= now) {
      int32_t clean = orc_detector_window_masked(det, win_samples, win_busy,
                                                 (policy == 1 && proto == ORC_BSP) ? active : NULL, flag);
      int32_t any = 0;
      for (int32_t q = 0; q < n; q++) {
        any |= flag[q];
        win_samples[q] = 0.0;
        win_busy[q] = 0.0;
      }
      next_window += D;
      windows++;
      if (policy == 1) {                                             /* elastic */
        if (proto == ORC_BSP && any && bsp_samples < quota) {
          int32_t left = 0;
          for (int32_t q = 0; q < n; q++) left += active[q] && !flag[q];
          if (left >= 1) {                                           /* a non-straggler must remain */
            int32_t m = 0;
            for (int32_t q = 0; q < n; q++) {
              if (flag[q]) active[q] = 0;
              if (active[q]) ids[m++] = q;
            }
            n_active = m;
            if (st) orcf_set_members(st, ids, m);
            if (nlog < cap) {
              log5[5 * nlog + 0] = now; log5[5 * nlog + 1] = version; log5[5 * nlog + 2] = ORC_BSP;
              log5[5 * nlog + 3] = 3;   log5[5 * nlog + 4] = n_active;
            }
            nlog++;
          }
        }
      } else if (policy == 2) {
        /* no straggler policy */
      } else if (proto == ORC_BSP && any && bsp_samples < quota) {   /* P:1421 straggler during BSP */
        LOG_SWITCH(ORC_ASP, 1);
        BEGIN_ASP();
      } else if (proto == ORC_ASP && clean && bsp_samples < quota) { /* P:1421 clean and BSP unfinished */
        LOG_SWITCH(ORC_BSP, 2);
        for (int32_t q = 0; q < n; q++) {
          if (st) orcf_asp_push(st, q, g[0], base[q], NULL);          /* late: rejected, counted as dropped */
          steps[q]++;
          dropped++;
        }
      }
    }
  }
#undef STEP_LEN
#undef LOG_SWITCH
#undef BEGIN_ASP
  res7[0] = bsp_steps; res7[1] = asp_pushes; res7[2] = dropped; res7[3] = now; res7[4] = version;
  res7[5] = windows; res7[6] = nlog;
  for (int32_t j = 0; j < n; j++) free(g[j]);
  free(g); free(steps); free(base); free(finish); free(length); free(win_samples); free(win_busy); free(flag);
  free(ver);
  free(ids);
  free(active);
  orc_detector_free(det);
  return nlog;
}

/* ------------------------------------------------------------------------------------------------------------
 * Dynamic switching criterion (draft design P:226-243; reading C18: g is the per-sample MEAN, lag x_{i-k}).
 * Written literally: per-sample gradients are materialised, then
 *   g = (1/B) sum_b grad_b,  Delta = g - g_prev,
 *   sigma = 1/(B |Delta|) * sqrt( sum_b [Delta^T (grad_b - g)]^2 )
 * per_sample: B x P row-major. sigma = 0 when |Delta| = 0. */
void orc_criterion(const double *per_sample, int32_t B, int64_t P, const double *g_prev, double *norm_delta,
                   double *sigma) {
  double *g = (double *)calloc((size_t)P, sizeof(double));
  double *delta = (double *)malloc((size_t)P * sizeof(double));
  for (int32_t b = 0; b < B; b++)
    for (int64_t k = 0; k < P; k++) g[k] += per_sample[(int64_t)b * P + k];
  for (int64_t k = 0; k < P; k++) g[k] /= (double)B;
  double nd2 = 0.0;
  for (int64_t k = 0; k < P; k++) {
    delta[k] = g[k] - g_prev[k];
    nd2 += delta[k] * delta[k];
  }
  double ss = 0.0;
  for (int32_t b = 0; b < B; b++) {
    double proj = 0.0;                                  /* Delta^T (grad_b - g) */
    for (int64_t k = 0; k < P; k++) proj += delta[k] * (per_sample[(int64_t)b * P + k] - g[k]);
    ss += proj * proj;
  }
  *norm_delta = sqrt(nd2);
  *sigma = nd2 > 0.0 ? sqrt(ss) / ((double)B * sqrt(nd2)) : 0.0;
  free(g);
  free(delta);
}

/* Per-sample gradients of the softmax-regression loss -log p_{y_b}(x_b W): grad_b[i, c] = x_b[i] (p_b[c] - [c == y_b]).
 * out: B x (d*C) row-major, fp64. */
void orc_softmax_per_sample(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const double *W,
                            double *out) {
  double *z = (double *)malloc((size_t)C * sizeof(double));
  for (int32_t b = 0; b < B; b++) {
    const float *x = X + (int64_t)b * d;
    for (int32_t c = 0; c < C; c++) {
      double acc = 0.0;
      for (int32_t i = 0; i < d; i++) acc += (double)x[i] * W[(int64_t)i * C + c];
      z[c] = acc;
    }
    double m = z[0];
    for (int32_t c = 1; c < C; c++) if (z[c] > m) m = z[c];
    double den = 0.0;
    for (int32_t c = 0; c < C; c++) den += exp(z[c] - m);
    for (int32_t c = 0; c < C; c++) {
      double r = exp(z[c] - m) / den - (c == y[b] ? 1.0 : 0.0);
      for (int32_t i = 0; i < d; i++) out[(int64_t)b * d * C + (int64_t)i * C + c] = (double)x[i] * r;
    }
  }
  free(z);
}

/* "we switch from BSP to ASP at the first time i when |Delta_i| < c sigma_i ... (or perhaps once this criterion is
 * satisfied for some number T steps in a row)". |Delta| = 0 counts as satisfied. */
int32_t orc_criterion_observe(int32_t *run, double norm_delta, double sigma, double c, int32_t T) {
  int32_t satisfied = norm_delta == 0.0 || norm_delta < c * sigma;
  *run = satisfied ? *run + 1 : 0;
  return *run >= T;
}
