/*
 * oracle.h — plain, slow, single-threaded CPU oracle for the Sync-Switch sharded-PS synchronization path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing on the product path (paper_2104_08364_b200/, include/) may include, link,
 * load or execute anything under oracle/. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may. The oracle shares no code, header, table or generator with the CUDA path.
 *
 * Citation shorthand: P:L = PAPER.md line L (arXiv 2104.08364 source), S:L = SPEC.md line L, SV = SURVEY.md.
 * Every function states the passage it follows; DESIGN.md §3 lists every reading taken where the paper is silent.
 *
 * Status values (numerically equal to the C-ABI's by specification, SV §8b; defined independently here):
 */
#ifndef SYNCSWITCH_ORACLE_H
#define SYNCSWITCH_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_E_INVAL = 1,
  ORC_E_STATE = 2,
  ORC_E_PROTOCOL = 3,
  ORC_E_BARRIER = 4,
  ORC_E_CAUSALITY = 5,
  ORC_E_DIVERGED = 6
};
enum { ORC_BSP = 0, ORC_ASP = 1 };

/* ---- shard layout ("divide the model parameters into different shards, each shard managed by one PS
 * instance"; P:1071 #PS = #workers; SV §8a a1) ---- */
int64_t orc_shard_pad(int64_t P, int32_t S);                  /* ceil(ceil(P/S)/32)*32 */
void orc_shard_offsets(int64_t P, int32_t S, int64_t *off);   /* off[s] = min(s*pad, P), S+1 entries */
int32_t orc_shard_owner(int32_t s, int32_t S, int32_t G);     /* floor(s*G/S) */
int32_t orc_worker_host(int32_t j, int32_t n, int32_t G);     /* floor(j*G/n) */

/* ---- learning rate (P:1600 schedule; P:1473 eta_BSP = n*eta; P:1490 eta_ASP = eta/sqrt(n)) ---- */
double orc_lr_factor(int64_t version, const int64_t *bounds, const float *factors, int32_t nb);
float orc_lr(float eta, double factor, int32_t proto, int32_t n, int32_t asp_rule);
/* Table I: workload-preserving remap. s = s_num/s_den is the BSP share of W samples.
 * Writes bsp_steps, asp_steps and nb remapped boundaries (version coordinate). Returns 0, or -1 when a
 * quantity is not an integer. */
int32_t orc_table1(int64_t W, int64_t B, int64_t N, int64_t s_num, int64_t s_den, const int64_t *Wb, int32_t nb,
                   int64_t *bsp_steps, int64_t *asp_steps, int64_t *bounds_out);

/* ---- protocol state machine (BSP P:1091-1093, ASP P:1099-1103, switch P:1531/P:280) ----
 * Two precisions with identical semantics: orcf_* in fp32 (parity with the GPU) and orcd_* in fp64 (identities). */
typedef struct orc_f orc_f;
typedef struct orc_d orc_d;

#define ORC_DECLARE(SUF, REAL)                                                                                   \
  orc_##SUF *orc##SUF##_new(const REAL *params, int64_t P, int32_t S, int32_t n, float lr, float mu, int32_t *st); \
  void orc##SUF##_free(orc_##SUF *o);                                                                            \
  int32_t orc##SUF##_set_lr_schedule(orc_##SUF *o, const int64_t *bounds, const float *factors, int32_t nb);     \
  int32_t orc##SUF##_set_lr_policy(orc_##SUF *o, int32_t asp_rule, float weight_decay);                          \
  int32_t orc##SUF##_set_momentum_policy(orc_##SUF *o, int32_t rule, int64_t samples_per_epoch, int64_t batch);   \
  int32_t orc##SUF##_set_nesterov(orc_##SUF *o, int32_t on);                                                    \
  int32_t orc##SUF##_set_members(orc_##SUF *o, const int32_t *workers, int32_t count);                           \
  int32_t orc##SUF##_bsp_step(orc_##SUF *o, const REAL *const *grads, const int32_t *workers,                     \
                              const int64_t *versions, int32_t n_local);                                         \
  int32_t orc##SUF##_asp_push(orc_##SUF *o, int32_t worker, const REAL *grad, int64_t version, int64_t *stale);  \
  int32_t orc##SUF##_pull(orc_##SUF *o, int32_t worker, REAL *dst, int64_t *version_out);                        \
  int32_t orc##SUF##_switch(orc_##SUF *o, int32_t proto, int64_t at_step);                                       \
  int32_t orc##SUF##_read_params(orc_##SUF *o, REAL *dst);                                                       \
  int32_t orc##SUF##_read_velocity(orc_##SUF *o, REAL *dst);                                                     \
  int32_t orc##SUF##_stats(orc_##SUF *o, int64_t *version, int32_t *proto, uint64_t *hist, int32_t hist_len,     \
                           uint64_t *dropped);                                                                   \
  int64_t orc##SUF##_log_len(orc_##SUF *o);                                                                      \
  int32_t orc##SUF##_log_get(orc_##SUF *o, int64_t i, int64_t *rec4);                                            \
  float orc##SUF##_current_lr(orc_##SUF *o, int32_t proto);

ORC_DECLARE(f, float)
ORC_DECLARE(d, double)

/* ---- seeded synthetic inputs, written from SV §8d (independent of the CUDA generator) ---- */
uint64_t orc_splitmix64(uint64_t x);
/* g[i - i0] for i in [i0, i0+count): key = (j<<56) ^ (k<<30) ^ i; h = splitmix64(seed ^ key);
 * g = ((h>>40)*2^-24 - 0.5)*2^-6 */
void orc_synth_grad(uint64_t seed, int32_t j, int64_t k, int64_t i0, int64_t count, float *out);

/* Integer-tick arrival schedule (SV §8c C7): worker j's k-th push at t_{j,k} = t_{j,k-1} + T_j(t_{j,k-1}) + d_{j,k},
 * t_{j,0} = 0 (first pull); each push is followed immediately by that worker's pull; global order by (t, j).
 * T_j(t) = period[j] * slow_factor if j == slow_worker and slow_t0 <= t < slow_t1, else period[j].
 * d_{j,k} = (splitmix64(seed ^ (j<<32) ^ k) mod (2J+1)) - J.
 * Writes the first n_push pushes (events: kind 0 = push, 1 = pull; worker; tick) into ev_* (capacity 2*n_push
 * + n for the initial pulls). Returns the number of events written. */
int64_t orc_schedule(int32_t n, const int64_t *period, int64_t jitter, uint64_t seed, int32_t slow_worker,
                     int64_t slow_factor, int64_t slow_t0, int64_t slow_t1, int64_t n_push, int32_t *ev_kind,
                     int32_t *ev_worker, int64_t *ev_tick);

/* ---- toy model (SV config 1): softmax regression, fp64. W is d x C row-major (P = d*C). ----
 * loss = -(1/B) sum_b log p_{b,y_b}; grad = X^T (p - Y) / B. */
double orc_softmax_loss_grad(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const double *W,
                             double *grad);

/* ---- straggler detector and greedy policy ---- */
typedef struct orc_detector orc_detector;
orc_detector *orc_detector_new(int32_t n, int32_t K);
void orc_detector_free(orc_detector *dt);
/* One detection window: S_k = samples[k] / busy[k]; flag S_k < mean - sigma_pop. Writes straggler[k] = 1 if
 * worker k has been flagged for K consecutive windows. Returns 1 if no worker was flagged for the last K windows
 * ("cluster free of stragglers", SV C15), else 0. */
int32_t orc_detector_window(orc_detector *dt, const double *samples, const double *busy, int32_t *straggler);
/* Same over the workers with mask[k] != 0 (elastic policy): others are not measured, not flagged, counters reset. */
int32_t orc_detector_window_masked(orc_detector *dt, const double *samples, const double *busy, const uint8_t *mask,
                                   int32_t *straggler);

/* ---- online straggler scenario (config 4): greedy policy over the detector ----
 * policy 0 greedy, 1 elastic, 2 none. st: an orcf_* state with n workers (NULL: dry run).
 * Writes up to cap records {tick, version, to, reason, members} to log5 (reason 3: elastic removal) and {bsp_steps, asp_pushes, dropped, end_tick, version, windows, n_switches} to res7. Returns n_switches. */
int64_t orc_scenario_run(orc_f *st, int64_t P, int32_t n, int64_t B, int64_t W, int64_t q_num, int64_t q_den,
                         int64_t period, int64_t jitter, uint64_t sched_seed, uint64_t grad_seed, int32_t slow_worker,
                         int64_t slow_factor, int64_t slow_t0, int64_t slow_t1, int64_t D, int32_t K,
                         int32_t policy, int64_t *log5, int32_t cap, int64_t *res7);

/* ---- dynamic switching criterion (reading C18), fp64, literal ---- */
void orc_criterion(const double *per_sample, int32_t B, int64_t P, const double *g_prev, double *norm_delta,
                   double *sigma);
void orc_softmax_per_sample(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const double *W,
                            double *out);
int32_t orc_criterion_observe(int32_t *run, double norm_delta, double sigma, double c, int32_t T);

#ifdef __cplusplus
}
#endif
#endif
