/*
 * syncswitch.h — C-ABI of the B200-native Sync-Switch synchronization path (arXiv 2104.08364).
 *
 * The library (`libsyncswitch.so`, built from paper_2104_08364_b200/csrc/) implements the collocated, sharded
 * parameter-server synchronization step of Sync-Switch — BSP, ASP and the runtime protocol switch — with
 * hand-written sm_100a CUDA kernels and NCCL over NVLink. Citation shorthand: P:L = PAPER.md line L, S:L = SPEC.md
 * line L, SV = SURVEY.md, DESIGN = DESIGN.md at the repo root.
 *
 * Conventions (SV §8b):
 *  - Every call returns an ss_status; none throws or aborts. On error nothing is applied ("errors never partially
 *    apply"); ss_last_error() describes the most recent error of that context.
 *  - Integer protocol results (versions, staleness, histogram, dropped count) are computed on the host and are
 *    final when the call returns. Device data movement is stream-ordered on the context's stream and may be
 *    batched lazily (ASP windows); it is complete after ss_sync().
 *  - Pointers documented "host or device" may point to device memory (cudaMalloc / torch CUDA tensors), pinned or
 *    pageable host memory; host data is staged through a ring of device buffers on dedicated H2D / D2H copy streams
 *    ordered by events, so transfers in both directions overlap the kernels.
 *  - Buffers passed to a call are BORROWED until the next ss_sync() returns (the library may read/write them
 *    lazily); params passed to ss_init are COPIED. The caller keeps ownership of every buffer it passes.
 *  - A context is not thread-safe: one thread per context, calls in program order.
 *  - SS_E_DIVERGED is sticky: once a non-finite parameter or momentum value is produced (detected on the device,
 *    surfaced no later than the next ss_sync), every later call returns it ("failed training").
 *  - Multi-GPU (one process per GPU): after ss_init_dist, ss_bsp_step, ss_asp_push, ss_pull, ss_asp_replay,
 *    ss_switch, ss_sync and ss_read_params are collective: every rank makes the same call sequence (SPMD).
 *    Protocol errors (versions, barrier sets, protocol state) are decided on host state every rank shares, so they
 *    fail on every rank alike. An argument only one rank sees (the hosting rank's gradient or pull destination) can
 *    fail on that rank alone: the other ranks' fused kernels then give up after 10 s and report SS_E_CUDA at their
 *    next ss_sync (NCCL mode: the collective blocks) — validate such arguments before the call on every rank.
 */
#ifndef SYNCSWITCH_H
#define SYNCSWITCH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ss_ctx ss_ctx;

typedef enum { SS_BSP = 0, SS_ASP = 1 } ss_protocol;

typedef enum {
  SS_OK = 0,
  SS_E_INVAL = 1,     /* null pointer, n_params < 1, shards < 1, workers < 1 or > 256, lr <= 0, momentum not in
                         [0,1), worker id out of range, bad schedule, unsupported layout                           */
  SS_E_STATE = 2,     /* call invalid in the current protocol (bsp_step under ASP; asp_push under BSP — a late
                         in-flight push after an ASP->BSP switch lands here and is counted in dropped_pushes,
                         S:276), a second pending switch, or a multi-GPU call out of order                         */
  SS_E_PROTOCOL = 3,  /* BSP: missing or duplicate worker in a superstep                                   */
  SS_E_BARRIER = 4,   /* BSP: a gradient's base version != current version                                 */
  SS_E_CAUSALITY = 5, /* ASP: base version > current version                                              */
  SS_E_DIVERGED = 6,  /* non-finite value produced; sticky                                          */
  SS_E_CUDA = 7,      /* CUDA runtime error (message in ss_last_error)                                             */
  SS_E_NCCL = 8,      /* NCCL error                                                                               */
  SS_E_OOM = 9        /* device allocation failed                                                                  */
} ss_status;

/* ============================================================================================================
 * Lifecycle
 * ============================================================================================================ */

/* Create the synchronization state on the current CUDA device (P:1071 collocated PS per worker; P:15 shards).
 *   params    host or device fp32[n_params], COPIED: the initial model w ("w is a large vector distributed
 *             into parameter servers").
 *   n_shards  S >= 1 PS shards: contiguous, equal, padded to 32 floats (128 B); shard s covers
 *             [min(s*pad, P), min((s+1)*pad, P)) with pad = ceil(ceil(P/S)/32)*32 (SV §8a a1).
 *   n_workers n in [1, 256] ("equal numbers of PSs and workers" is the paper's default, not required).
 *   lr        base learning rate eta > 0; momentum mu in [0, 1) ("SGD with momentum of 0.9").
 * Default policy: protocol BSP at version 0 ("start with BSP"), BSP lr = n*eta, ASP lr = eta/sqrt(n)
 * (P:1490), no lr decay, weight decay 0. Momentum v = 0. Errors: SS_E_INVAL, SS_E_OOM, SS_E_CUDA (*out = NULL). */
ss_status ss_init(ss_ctx **out, const float *params, int64_t n_params, int32_t n_shards, int32_t n_workers,
                  float lr, float momentum);

/* Join `world` ranks (one process per GPU, one context per process) into one sharded PS. Collective; call once
 * before the first step. nccl_unique_id: the 128-byte ncclUniqueId created by rank 0 and broadcast by the caller.
 * Shard s is owned by rank floor(s*world/S); worker j is hosted on rank floor(j*world/n) (SV §8a a1).
 * Requires S % world == 0 (equal owner regions for reduce-scatter / all-gather). Errors: SS_E_INVAL, SS_E_STATE
 * (already stepped or already distributed), SS_E_NCCL. */
ss_status ss_init_dist(ss_ctx *ctx, int32_t rank, int32_t world, const void *nccl_unique_id);

/* Multi-GPU exchange implementation (collective; every rank passes the same mode):
 *   0  NCCL: BSP = local pre-sum -> ncclReduceScatter -> owner bsp_update -> ncclAllGather; ASP windows = grouped
 *      ncclSend/ncclRecv of gradient slices to owners and snapshot slices to pullers.
 *   1  fused peer memory, exact (default): CUDA-IPC-mapped buffers over NVLink/NVSwitch. A scatter kernel stores each
 *      hosted gradient's owner slices into the owners' inboxes; the owner kernel sums the n worker slices in
 *      ascending worker order (bit-identical to the single-GPU result), updates w and v, and stores the new slice into
 *      every rank's replica (BSP) or each pull's snapshot slice into the puller's buffer (ASP). Cross-GPU ordering by
 *      release/acquire flags inside the kernels (bounded waits: a missing peer yields SS_E_CUDA at ss_sync, never a
 *      hang). At most 8 ranks.
 *   2  fused peer memory, pre-summed: as 1, but each rank first sums its hosted workers and sends one slice per
 *      owner (fewer NVLink bytes when n > world; summation order: ascending within a rank, then ascending ranks).
 *   3  fused pull (BSP supersteps in ONE kernel per rank): every hosted gradient sits in the
 *      rank's exported gradient buffer of its worker (ss_grad_buffer: zero copy; any other buffer — device or host —
 *      is copied into it on the context's stream first); each owner loads its region of every member's gradient
 *      (hosted ones from local HBM, the others over NVLink), sums them in ascending worker order (bit-identical to
 *      one GPU), updates w and v and stores the new slice into every replica, between a cross-GPU barrier at kernel
 *      entry and one at exit. ASP windows run as in mode 1. Moves the fewest NVLink bytes when every rank hosts at
 *      most one worker (n <= world, the paper's one-PS-per-worker-node layout).
 * In modes 1, 2 and 3 the BSP broadcast of the updated slices uses P2P stores at every world size; environment variable
 * SS_NVLS=1 switches it to NVSwitch multicast (NVLS, one multimem.st per element reaches every replica; opt-in: no
 * speed-up measured at 2 or 4 GPUs). Errors: SS_E_INVAL. */
ss_status ss_set_fused(ss_ctx *ctx, int32_t mode);

/* The exchange in effect: *mode = the ss_set_fused mode (0 on a single GPU), *nvls = 1 once the fused path has set up
 * its NVSwitch multicast replica (decided collectively at the first fused call), else 0. Any output may be NULL.
 * Errors: none besides a diverged context. */
ss_status ss_get_exchange(ss_ctx *ctx, int32_t *mode, int32_t *nvls);

/* Fused multi-GPU mode: the CUDA-IPC-mapped pull buffer (device fp32[P_pad], owned by the context, valid until
 * ss_destroy) of a worker hosted on this rank. Owners store each pull's snapshot slices into it over NVLink; passing
 * it as ss_pull's dst makes the pull zero-copy (otherwise the snapshot is copied from it into dst). Collective on
 * first use. Errors: SS_E_INVAL (worker not hosted here), SS_E_STATE (single GPU or NCCL mode). */
ss_status ss_pull_buffer(ss_ctx *ctx, int32_t worker, float **out);

/* P:1072 ("push the computed gradients to all PSs"), SV §8(f) NEXT-1 (the owner loads the peers' gradient slices).
 * Fused multi-GPU mode: the CUDA-IPC-mapped gradient buffer (device fp32[P_pad], owned by the context, valid until
 * ss_destroy; the padding past n_params must stay 0) of a worker hosted on this rank. In mode 3 owners load their
 * region of it over NVLink during a superstep: a worker that writes its gradient here and passes this pointer to
 * ss_bsp_step saves the copy-in. Like every gradient it is BORROWED by the superstep until ss_sync. Collective on
 * first use. Errors: SS_E_INVAL (worker not hosted here), SS_E_STATE (single GPU or NCCL mode). */
ss_status ss_grad_buffer(ss_ctx *ctx, int32_t worker, float **out);

/* Fills the 128-byte buffer with a fresh ncclUniqueId (rank 0 calls this, then broadcasts it). */
ss_status ss_nccl_unique_id(void *out128);

/* Releases every device buffer, the stream and the communicator. Flushes pending work first. NULL is a no-op. */
void ss_destroy(ss_ctx *ctx);

/* Human-readable description of the last error on ctx (never NULL; "" when none). */
const char *ss_last_error(const ss_ctx *ctx);

/* ============================================================================================================
 * Policy (configuration policy P:1472-1474, schedule P:1600, Table I)
 * ============================================================================================================ */

/* Piecewise-constant lr decay in the VERSION coordinate (Table I's "total steps"): the factor is 1 before
 * boundaries[0] and factors[i] from boundaries[i] on (multipliers of the base lr, not cumulative).
 * boundaries strictly ascending, >= 0; factors > 0; n in [0, 64]. Copied. Errors: SS_E_INVAL. */
ss_status ss_set_lr_schedule(ss_ctx *ctx, const int64_t *boundaries, const float *factors, int32_t n);

/* asp_rule: 0 -> eta_ASP = eta/sqrt(n), 1 -> eta/n, 2 -> eta. weight_decay lambda >= 0: f(w) = lambda*w
 * added to each gradient at apply time at the PS's current w ("g11 + f(w0)"). Errors: SS_E_INVAL. */
ss_status ss_set_lr_policy(ss_ctx *ctx, int32_t asp_rule, float weight_decay);

/* Post-switch momentum policy for ASP pushes (SV §8(f) NEXT-4; "setting the momentum to 0 ...
 * to 1/n ... ramping up the momentum based on 2^i/n ... based on i/n where i is the number of epochs after switching.
 * Both (iii) and (iv) will stop the ramp up once the momentum reaches the original value used by BSP"):
 *   rule 0: same momentum as BSP (default; the paper's chosen policy)   rule 1: 0   rule 2: 1/n
 *   rule 3: 2^i/n   rule 4: i/n,   all capped at the BSP momentum (DESIGN reading C24),
 * with i = floor(pushes since the last switch to ASP * batch / samples_per_epoch). Computed per push in double and
 * rounded to fp32 once; BSP supersteps always use the BSP momentum. Errors: SS_E_INVAL. */
ss_status ss_set_momentum_policy(ss_ctx *ctx, int32_t rule, int64_t samples_per_epoch, int64_t batch);

/* Nesterov momentum (SV §8(f) NEXT-4; the paper never names the momentum form, reading C1 takes the accumulator form
 * of the prototype's TF MomentumOptimizer; this switch is that optimizer's use_nesterov variant, DESIGN
 * reading C28): on = 1 -> v = mu*v + g, w = w - eta*(g + mu*v) with each product-sum one fused multiply-add
 * (fma(mu, v, g) then fma(-eta, ., w)); on = 0 (default) -> w = w - eta*v. Applies to BSP supersteps and ASP pushes
 * applied after the call (a pending ASP window is flushed first). Errors: SS_E_INVAL (on not 0/1). */
ss_status ss_set_nesterov(ss_ctx *ctx, int32_t on);

/* BSP barrier set for the elastic straggler policy (SV §8(f) NEXT-2; "removes any detected stragglers from the
 * current cluster so as to complete the specified amount of BSP training free of stragglers. Once the designated BSP
 * workload is fulfilled, it will then restore the cluster size"). workers: `count` distinct ids in [0, n). Later
 * BSP supersteps expect exactly these workers' gradients; the aggregate is their mean in ascending worker order and
 * the BSP lr is count*eta (configuration policy re-derived for the smaller cluster). ASP is unaffected.
 * Restore with all n ids. Collective when distributed. Errors: SS_E_INVAL (empty, duplicate, out of range). */
ss_status ss_set_members(ss_ctx *ctx, const int32_t *workers, int32_t count);

/* lr used for the next update under `protocol`: (float)((double)eta * factor(version) * scale(protocol)). */
ss_status ss_current_lr(ss_ctx *ctx, int32_t protocol, float *lr_out);

/* ============================================================================================================
 * The synchronization path
 * ============================================================================================================ */

/* BSP superstep (Fig. 3: gradients are aggregated at a barrier, then the model is updated).
 *   grads[i]    host or device fp32[n_params]: the gradient of worker workers[i] (BORROWED until ss_sync; host
 *               memory is staged on a copy stream). Device pointers should be 16-byte aligned (the fused multi-GPU
 *               path requires it; single GPU falls back to a scalar kernel otherwise).
 *   versions[i] the base version that gradient was computed on; must equal the current version.
 *   n_local     number of gradients supplied: exactly the BSP members (all n unless ss_set_members shrank the
 *               set), each once; multi-GPU: exactly the members hosted on this rank.
 * Computes g = (sum_{members, ascending} g_j) / m (+ lambda*w), v = mu*v + g, w = w - eta_BSP*v over every shard
 * (m = number of members; kernel bsp_update; G > 1 per ss_set_fused: NCCL reduce-scatter / all-gather, or the
 * fused peer-memory scatter -> owner update -> broadcast), then version += 1 and every worker's base version =
 * version; one staleness-0 record per member.
 * Errors: SS_E_STATE (protocol is ASP), SS_E_PROTOCOL (missing/duplicate/non-member worker), SS_E_BARRIER,
 * SS_E_INVAL. */
ss_status ss_bsp_step(ss_ctx *ctx, const float *const *grads, const int32_t *workers, const int64_t *versions,
                      int32_t n_local);

/* ASP push (w1 = w0 - eta_t(g11 + f(w0)) applied on arrival). grad: host or device fp32[n_params] of
 * `worker`, BORROWED until ss_sync (multi-GPU: non-NULL only on the rank hosting `worker`; NULL elsewhere).
 * version: the worker's base version (from its last ss_pull). Returns *staleness_out = current - version
 * immediately, then version += 1. The update itself is applied by the asp_replay kernel when the
 * replay window is flushed: when it holds ss_set_window events (pushes and pulls count), or at ss_sync,
 * ss_read_params, a switch taking effect, ss_bsp_step, ss_set_window/ss_set_fused/ss_set_lr_policy, capture end.
 * Errors: SS_E_STATE (protocol is BSP; counted in dropped_pushes), SS_E_CAUSALITY, SS_E_INVAL. */
ss_status ss_asp_push(ss_ctx *ctx, int32_t worker, const float *grad, int64_t version, int64_t *staleness_out);

/* Pull ("a worker will first pull model parameters from all PSs"). dst: host or device fp32[n_params]
 * (BORROWED until ss_sync). NULL = version only (single GPU); multi-GPU: every pull moves data, so dst must be
 * non-NULL on the rank hosting `worker` and NULL elsewhere. A pull is an event of the replay window: dst receives the
 * parameters after exactly the pushes that precede this call (on every shard), valid after ss_sync. *version_out =
 * current version; it becomes the worker's base version. Errors: SS_E_INVAL. */
ss_status ss_pull(ss_ctx *ctx, int32_t worker, float *dst, int64_t *version_out);

/* Switch to `protocol` when the version reaches at_step (at_step <= current: now). w, v and version are carried
 * over bit-identically (P:280 momentum carried over; P:1531 the prototype's checkpoint/relaunch becomes an in-place
 * flip). ASP -> BSP drops in-flight pushes and sets every worker's base version to the switch version (every worker
 * implicitly pulls). One pending switch at a time. Errors: SS_E_INVAL, SS_E_STATE (a switch is already pending). */
ss_status ss_switch(ss_ctx *ctx, int32_t protocol, int64_t at_step);

/* Batched ASP fast path: identical semantics to the equivalent ss_asp_push / ss_pull call sequence (kind 0 = push
 * with grad and version; kind 1 = pull into dst, its version is written to staleness_out[i]). Stops at the first
 * failing event and returns its status; events before it are applied. staleness_out: int64[n_ev] or NULL. */
typedef struct {
  int32_t kind;    /* 0 push, 1 pull */
  int32_t worker;
  int64_t version; /* push: base version */
  const float *grad;
  float *dst;
} ss_event;
ss_status ss_asp_replay(ss_ctx *ctx, const ss_event *ev, int64_t n_ev, int64_t *staleness_out);

/* Flush the pending window, wait for the context's streams, surface asynchronous errors (SS_E_DIVERGED; SS_E_CUDA,
 * including a fused-path cross-GPU wait that timed out). Not allowed while capturing a graph (SS_E_STATE). */
ss_status ss_sync(ss_ctx *ctx);

/* SV §8b ("device data movement is stream-ordered and may be lazily batched"); P:1072 (a worker computes its next
 * gradient from the parameters it pulled).
 * Issue the device work of the calls accepted so far (the pending window, including one-GPU supersteps deferred into
 * it) on the context's stream, without waiting. A caller whose next inputs depend on these results (a worker that
 * computes its next gradient from a pulled snapshot, or from the parameters after a superstep) flushes, then orders
 * its own stream after the context's (ss_wait_stream) — the window batching never reaches across such a dependency.
 * Buffers stay BORROWED until ss_sync. Collective when distributed. Errors: SS_E_DIVERGED, SS_E_CUDA, SS_E_NCCL. */
ss_status ss_flush(ss_ctx *ctx);

/* Copies the unpadded parameters w (fp32[n_params]) / momentum v to a HOST buffer (collective when distributed).
 * Flushes and synchronizes first. */
ss_status ss_read_params(ss_ctx *ctx, float *host_dst);
ss_status ss_read_velocity(ss_ctx *ctx, float *host_dst);

/* Protocol counters: current version, protocol, staleness histogram hist[0..hist_len) (BSP updates count as
 * staleness 0), pushes dropped at ASP->BSP switches. Any output may be NULL. */
ss_status ss_get_stats(ss_ctx *ctx, int64_t *version, int32_t *protocol, uint64_t *hist, int32_t hist_len,
                       uint64_t *dropped_pushes);

/* Applied-gradient log, one record per applied gradient in apply order: {worker, base version, staleness, version
 * at apply}. Writes min(cap, total) records to rec4 (int64[4*cap]); *total_out = number of records. */
ss_status ss_get_log(ss_ctx *ctx, int64_t *rec4, int64_t cap, int64_t *total_out);

/* ============================================================================================================
 * Execution control and instrumentation
 * ============================================================================================================ */

/* Maximum events (pushes + pulls) per ASP replay window, 1..64 (default 16). Flushes first. */
ss_status ss_set_window(ss_ctx *ctx, int32_t max_events);
/* The cudaStream_t all work of this context is ordered on (owned by the context). */
ss_status ss_get_stream(ss_ctx *ctx, void **stream_out);
/* Order the context's work after `stream` (cudaStream_t) — used when gradients are produced on another stream. */
ss_status ss_wait_stream(ss_ctx *ctx, void *stream);
/* CUDA-graph capture of one step (SV §8(d): latency-bound small models "with and without CUDA Graphs", G = 1..8).
 * Between ss_capture_begin and ss_capture_end, the calls run their host logic as usual but their device work is
 * recorded into a graph instead of executing; ss_capture_end instantiates it and launches it once (so the captured
 * step has happened on both sides) and returns the step's version delta. ss_capture_replay(K) launches the graph K
 * more times and applies the step's host-state deltas K times (versions, base versions, staleness histogram and
 * log with shifted versions, dropped pushes). Replay requires the step to leave the protocol state as it found it
 * (relative base versions, no pending switch, no queued window) and nothing baked into the kernels to change over
 * the replayed versions (no lr boundary inside, momentum rule 0). Buffers the step used stay BORROWED while a
 * graph exists. Calls that allocate (first use of host buffers) must not happen during capture: warm up first.
 * Multi-GPU: collective — every rank captures the same step and replays it the same number of times; run one
 * ordinary step first (the exchange buffers, peer mappings and NVLS replica are set up lazily). The fused kernels'
 * cross-GPU flag epochs come from a device-resident counter, so replays synchronise with fresh epochs.
 * Errors: SS_E_STATE, SS_E_CUDA. */
ss_status ss_capture_begin(ss_ctx *ctx);
ss_status ss_capture_end(ss_ctx *ctx, int64_t *version_delta);
ss_status ss_capture_replay(ss_ctx *ctx, int64_t times);

/* Kernel timing: when on, every launch of the path's kernels is bracketed by CUDA events on the context's stream;
 * ss_kernel_stats returns per-kernel launch count, total device milliseconds, algorithmic HBM bytes and algorithmic
 * bytes sent over NVLink by the fused multi-GPU path (kernel_id 0 = bsp_update, 1 = asp_replay, 2 = local_sum,
 * 3 = scatter / scatter_sum). Any output may be NULL. Reading synchronizes. */
ss_status ss_profile(ss_ctx *ctx, int32_t on);
ss_status ss_kernel_stats(ss_ctx *ctx, int32_t kernel_id, int64_t *launches, double *total_ms, double *bytes,
                          double *nvlink_bytes);

/* ============================================================================================================
 * Seeded synthetic inputs and the toy model (SV §8d; kernels synth_grad and softmax_grad)
 * ============================================================================================================ */

/* dst[t] = g(seed, j, k, i0 + t) for t in [0, count): key = (j<<56) ^ (k<<30) ^ i, h = splitmix64(seed ^ key),
 * g = ((h>>40)*2^-24 - 0.5)*2^-6 (exact in fp32, uniform in [-1/128, 1/128)). dst: device fp32[count];
 * stream: cudaStream_t or NULL (legacy default stream). j < 256, k < 2^26, i0 + count <= 2^30. */
ss_status ss_synth_grad(uint64_t seed, int32_t j, int64_t k, int64_t i0, int64_t count, float *dst, void *stream);

/* Softmax regression (stands in for the worker's forward/backward): X device fp32[B*d] row-major,
 * y device int32[B], W device fp32[d*C] row-major (P = d*C). grad = X^T (softmax(XW) - onehot(y)) / B into device
 * fp32[d*C]; *loss_dev (device fp32[1]) = mean cross-entropy. B <= 1024, C <= 32. */
ss_status ss_softmax_grad(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const float *W,
                          float *grad, float *loss_dev, void *stream);

/* Dynamic switching criterion for the toy model (SV §8(f) NEXT-3): computes the batch gradient at W,
 * g_out = X^T (softmax(XW) - Y) / B (device fp32[d*C]), Delta = g_out - g_prev (g_prev: device fp32[d*C], the batch
 * gradient k steps earlier on another batch, P:233-235 with reading C18), and writes stats (device fp32[2]) =
 * {|Delta|, sigma} with sigma = sqrt(sum_b [Delta^T (grad_b - g)]^2) / (B |Delta|) over the batch's per-sample
 * gradients grad_b (sigma = 0 when Delta = 0). The per-sample projections use the rank-one form
 * grad_b = x_b (x) (p_b - y_b); sums accumulate in fp64 in a fixed order. B in [2, 1024], C <= 32. */
ss_status ss_dynamic_criterion(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const float *W,
                               const float *g_prev, float *g_out, float *stats, void *stream);

/* ============================================================================================================
 * Control plane (host only; no GPU needed)
 * ============================================================================================================ */

/* Table I workload-preserving remap: BSP steps = W*s/(B*N), ASP steps = W/B - W*s/B with s = s_num/s_den;
 * boundary W_i (samples) -> W_i/(B*N) if W_i <= W*s, else W_i/B - W*s/B + W*s/(B*N) (DESIGN reading C11).
 * Errors: SS_E_INVAL when a quantity is not integral. */
ss_status ss_table1(int64_t W, int64_t B, int64_t N, int64_t s_num, int64_t s_den, const int64_t *Wb, int32_t nb,
                    int64_t *bsp_steps, int64_t *asp_steps, int64_t *bounds_out);

/* Seeded integer-tick arrival schedule (DESIGN reading C7): all n workers pull at t = 0; worker j's k-th push at
 * t_{j,k} = t_{j,k-1} + T_j(t_{j,k-1}) + d_{j,k}, immediately followed by its pull; global order by (t, j).
 * T_j(t) = period[j] * slow_factor when j == slow_worker and slow_t0 <= t < slow_t1; d_{j,k} =
 * (splitmix64(seed ^ (j<<32) ^ k) mod (2J+1)) - J. Writes n + 2*n_push events to kind/worker/tick (capacity
 * n + 2*n_push each); *n_out = events written. Errors: SS_E_INVAL (period <= J, n out of range). */
ss_status ss_schedule(int32_t n, const int64_t *period, int64_t jitter, uint64_t seed, int32_t slow_worker,
                      int64_t slow_factor, int64_t slow_t0, int64_t slow_t1, int64_t n_push, int32_t *kind,
                      int32_t *worker, int64_t *tick, int64_t *n_out);

/* Straggler detector: per window, S_k = samples[k]/busy[k]; worker k is flagged when S_k < mean - sigma
 * (population sigma) and is a straggler after K consecutive flagged windows; *clean_out = 1 when no worker was
 * flagged for the last K windows ("cluster free of stragglers"). */
typedef struct ss_detector ss_detector;
ss_status ss_detector_new(ss_detector **out, int32_t n, int32_t K);
ss_status ss_detector_window(ss_detector *dt, const double *samples, const double *busy, int32_t *straggler,
                             int32_t *clean_out);
/* Same over the workers with mask[k] != 0 only (elastic policy: removed workers are neither measured nor flagged;
 * their consecutive-window counters restart). mask NULL = all workers. */
ss_status ss_detector_window_masked(ss_detector *dt, const double *samples, const double *busy, const uint8_t *mask,
                                    int32_t *straggler, int32_t *clean_out);
void ss_detector_free(ss_detector *dt);

/* Multi-GPU routing plan (SV §8(a) a8/a10, §8(e)) of an ASP event sequence as rank `rank` of `world` executes it:
 * the sequence is cut into replay windows exactly as the runtime cuts them (max_window events; in fused mode also
 * before a second pull of the same worker), and each window yields, in issue order, phase-0 ops (gradient slice of a
 * push: hosting rank -> every other owner) and phase-1 ops (snapshot slice of a pull: every other owner -> hosting
 * rank). op 0 = send (fused: posted NVLink store), 1 = recv. offset/count: the slice [offset, offset+count) of the
 * full vector. Writes min(cap, total) ops; *n_ops = total, *n_windows = windows. Host only. Errors: SS_E_INVAL. */
typedef struct {
  int32_t window, phase, op, peer, event;
  int64_t offset, count;
} ss_route_op;
ss_status ss_route_plan(int32_t rank, int32_t world, int32_t n_workers, int32_t n_shards, int64_t n_params,
                        int32_t max_window, int32_t fused, const int32_t *kind, const int32_t *worker, int64_t n_ev,
                        ss_route_op *ops, int64_t cap, int64_t *n_ops, int32_t *n_windows);

/* Persistence rule of the dynamic criterion ("we switch from BSP to ASP at the first time i when
 * |Delta_i| < c sigma_i ... or once this criterion is satisfied for some number T steps in a row"): updates the
 * consecutive-satisfied count *run (|Delta| = 0 counts as satisfied) and returns 1 when it reaches T. */
int32_t ss_criterion_observe(int32_t *run, float norm_delta, float sigma, float c, int32_t T);

/* Greedy online policy: given the detector's verdict, the protocol and the BSP quota, returns the switch
 * to issue now: -1 none, SS_ASP (a straggler appeared during BSP), SS_BSP (cluster clean, ASP, BSP quota unmet). */
int32_t ss_greedy_decision(int32_t protocol, int32_t any_straggler, int32_t cluster_clean, int64_t bsp_done,
                           int64_t bsp_quota);

/* ============================================================================================================
 * Online straggler scenario (SV config 4; P:1410-1425 greedy policy, P:1416 transient <= 100 s)
 * ============================================================================================================
 * A discrete-event run in integer ticks (DESIGN reading C23). BSP supersteps last max_j T_j(t) + d_{j,k} ticks (the
 * barrier waits for the slowest worker; busy time excludes the wait); under ASP every worker pushes after T_j + d and
 * pulls at once (reading C7). Every detection window of `window_ticks` feeds the detector (samples B per completed
 * worker step, busy ticks) and the greedy policy: straggler under BSP -> switch to ASP now; cluster clean under ASP and
 * BSP quota unmet -> switch to BSP now (in-flight pushes then arrive late and are dropped). BSP samples reaching
 * W * quota_num / quota_den switch to ASP for good (timing policy); the run ends when W samples are processed.
 * Worker j's k-th gradient is synth_grad(grad_seed, j, k, ...). */
typedef struct {
  int32_t n_workers;
  int64_t batch;          /* B samples per worker step */
  int64_t total_samples;  /* W */
  int64_t quota_num, quota_den;
  int64_t period;         /* T ticks */
  int64_t jitter;         /* J */
  uint64_t sched_seed, grad_seed;
  int32_t slow_worker;    /* -1: none */
  int64_t slow_factor, slow_t0, slow_t1;
  int64_t window_ticks;   /* detection window D */
  int32_t K;              /* consecutive windows */
  int32_t policy;         /* 0: greedy; 1: elastic (stragglers leave the BSP barrier set until the
                             BSP quota is met, then all workers are restored and ASP runs the rest); 2: none */
} ss_scenario;
typedef struct {
  int64_t tick, version;
  int32_t to_protocol, reason; /* reason 0: BSP quota met (timing policy), 1: straggler (greedy), 2: clean (greedy),
                                  3: elastic removal of stragglers from the BSP set (no protocol change) */
  int32_t members;             /* BSP members after the event */
} ss_switch_event;
typedef struct {
  int64_t bsp_steps, asp_pushes, dropped, end_tick, version, windows;
  int32_t n_switches;
} ss_scenario_result;
/* ctx: a context with n_workers workers (its stream runs the kernels; collective when distributed), or NULL for a
 * host-only dry run of the same event sequence (no data). log: cap entries (nullable). Errors: SS_E_INVAL, and every
 * error of the protocol calls it issues. */
ss_status ss_scenario_run(ss_ctx *ctx, const ss_scenario *sc, ss_scenario_result *out, ss_switch_event *log,
                          int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* SYNCSWITCH_H */
