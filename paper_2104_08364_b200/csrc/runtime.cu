// runtime.cu — C-ABI runtime of the Sync-Switch synchronization path (include/syncswitch.h).
//
// Host side: shard map (SV §8a a1), version / staleness table and BSP barrier checks (a3, a7), ASP window batcher
// (a9-a10), switch controller (a11) and lr policy (a12). Device side: w replica [P_pad], momentum v of the owned
// region, a non-finite flag, gradient / snapshot staging. Multi-GPU: NCCL reduce-scatter -> bsp_update ->
// all-gather for BSP; grouped send/recv owner routing for ASP windows (SV §8e).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <unordered_set>
#include <vector>

#include "internal.h"
#include "nvls.h"
#include "plan.h"
#include "syncswitch.h"

namespace {

constexpr int kMaxSchedule = 64;

struct Ev {
  int32_t kind;         // 0 push, 1 pull, 2 BSP superstep (one GPU: BSP supersteps join the window, see ss_bsp_step)
  int32_t worker;
  const float *src;     // push: device gradient (full length; staged if the caller's was host memory);
                        //       nullptr on ranks not hosting the worker
  float *dst;           // pull: device destination (full length) on the hosting rank, else nullptr
  float *host_dst;      // pull into host memory: D2H from dst after the window
  int32_t slot = -1;    // staging slot behind dst (host destination), or -1
  float lr;             // push: eta_ASP at the push's (pre-increment) version
  float mu;             // push: momentum (post-switch momentum policy); BSP: momentum
  bool data;            // pull: moves parameters (false: version-only pull, G = 1)
  float divisor = 1.f;  // BSP: number of barrier workers
  int32_t src0 = 0, n_src = 0;   // BSP: gradients win_bsp_src[src0 .. src0 + n_src), ascending workers
};

struct KStat {
  int64_t launches = 0;
  double ms = 0.0, bytes = 0.0, nvbytes = 0.0;
};

struct Timed {
  cudaEvent_t a, b;
  int kernel;
  double bytes;    // algorithmic HBM bytes of the launch
  double nvbytes;  // algorithmic bytes the launch sends over NVLink (fused multi-GPU path)
};

}  // namespace

struct ss_ctx {
  // configuration
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t P = 0, pad = 0, P_pad = 0;
  int32_t S = 0, n = 0;
  std::vector<int64_t> off;
  float eta = 0.f, mu = 0.f, lam = 0.f;
  int32_t nesterov = 0;                // ss_set_nesterov
  int32_t asp_rule = 0;
  int32_t mom_rule = 0;                // post-switch momentum policy: 0 same mu, 1 zero, 2 1/n, 3 2^i/n, 4 i/n
  int64_t mom_epoch_samples = 1, mom_batch = 1;
  int64_t asp_since = 0;               // version at which the last switch to ASP took effect
  std::vector<uint8_t> member;         // BSP barrier set (elastic policy); all workers by default
  int32_t n_members = 0;
  std::vector<int64_t> bounds;
  std::vector<float> factors;
  // distribution
  int32_t rank = 0, world = 1;
  ss::Layout L;                        // shard layout / ownership (plan.h)
  ncclComm_t comm = nullptr;
  int64_t reg_len = 0;                 // padded owner region length (P_pad / world)
  std::vector<int64_t> real_lo, real_hi;  // per rank: real (unpadded) element range of its region
  // device state
  float *w = nullptr;                  // replica [P_pad]; authoritative on the owned region
  float *v = nullptr;                  // momentum of the owned region [reg_len]
  int *flag = nullptr;                 // non-finite flag
  int *health = nullptr;               // G > 1: [flag, barrier timeout] agreed over ranks at ss_sync
  float *sum_buf = nullptr;            // G > 1: local pre-sum [P_pad]
  float *rs_buf = nullptr;             // G > 1: reduce-scattered sum [reg_len]
  std::vector<float *> stage;          // full-length staging slots for host pointers (a ring, see stage_slot)
  int32_t stage_next = 0;              // ring cursor once the pool is full
  std::vector<int32_t> win_slots;      // slots taken by the pending window / superstep, released after its kernels
  // host<->device staging copies run on their own streams so PCIe traffic in both directions overlaps
  // the kernels and each other; per-slot events order reuse (slot_free) and consumption (slot_ready)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  std::vector<cudaEvent_t> slot_free, slot_ready;
  std::vector<uint8_t> slot_armed;     // slot_free has been recorded at least once
  std::vector<float *> rslot, sslot;   // G > 1: received gradient shards / snapshot shards per window event
  // protocol state (host; bit-exact with the oracle)
  int64_t version = 0;
  std::vector<int64_t> base;
  int32_t proto = SS_BSP;
  bool has_pending = false;
  int32_t pending_proto = SS_BSP;
  int64_t pending_at = 0;
  std::vector<uint64_t> hist;
  uint64_t dropped = 0;
  bool diverged = false;
  bool stepped = false;
  std::vector<int64_t> log;            // 4 per applied gradient
  // window batcher
  std::vector<Ev> win;
  std::vector<int32_t> win_kind, win_worker;   // the window's ASP events (push / pull) for the cut rule
  std::vector<const float *> win_bsp_src;      // gradients of the window's BSP events
  int32_t max_win = 16;
  // fused peer-memory path (G > 1): CUDA-IPC-mapped inboxes, replicas, pull buffers and flags
  int32_t fused_mode = 1;              // 0 NCCL, 1 fused exact (ascending workers), 2 fused pre-summed, 3 fused pull
  bool ipc_ready = false;
  int64_t inbox_slots = 0;
  float *inbox = nullptr;              // [bufs][inbox_slots][reg_len] gradient slices owned here, written by peers
  int32_t inbox_bufs = 1;              // 2: exchanges alternate between two inbox buffers (no end barrier needed)
  int64_t xchg = 0;                    // fused exchanges issued (selects the inbox buffer)
  float *pbuf = nullptr;               // [n_hosted][P_pad] pull buffers of hosted workers, written by owners
  float *gbuf = nullptr;               // [n_hosted][P_pad] gradient buffers of hosted workers, read by owners (mode 3)
  uint32_t *sigblk = nullptr;          // [0..7] inbound flags, [32] CTA counter, [64] timeout flag, [160] epoch counter
  float *peer_w[ss::kMaxPeers] = {}, *peer_inbox[ss::kMaxPeers] = {}, *peer_pbuf[ss::kMaxPeers] = {};
  float *peer_gbuf[ss::kMaxPeers] = {};
  uint32_t *peer_sig[ss::kMaxPeers] = {};
  std::vector<void *> opened;          // peer mappings to close
  ss::NvlsReplica nvls;                // NVSwitch multicast replica (w lives here when ready)
  bool nvls_tried = false;
  bool w_vmm = false;                  // w points into the NVLS replica (not cudaMalloc memory)
  char job_tag[48] = {0};              // names the NVLS fd socket: hash of the NCCL unique id + setup count
  uint32_t epoch = 0;
  uint32_t dev_epoch = 0;              // host mirror of the device epoch counter sigblk[kSigEpochBase] (peer_sync)
  int32_t first_hosted = 0, n_hosted = 0;
  // CUDA-graph capture of one step (ss_capture_*): device work + the host-state deltas it produced
  bool capturing = false;
  cudaGraphExec_t graph = nullptr;
  int64_t cap_v0 = 0, cap_dv = 0, cap_log0 = 0, cap_rel_since = 0;
  uint64_t cap_ddropped = 0;
  uint32_t cap_epoch0 = 0, cap_depoch = 0;   // fused-path flag epochs consumed by the captured step
  int64_t cap_xchg0 = 0;                     // fused exchanges issued before the capture
  std::vector<int64_t> cap_base0, cap_log;   // log records appended during the captured step
  // instrumentation
  unsigned long long *trace_dev = nullptr;   // SS_TRACE=<prefix>: 4 globaltimer stamps per fused launch
  int64_t trace_cap = 0;
  std::vector<int8_t> trace_kind;            // per recorded launch: 0 scatter, 1 scatter_sum, 2 bsp_update, 3 asp_replay
  std::string trace_path;
  bool prof = false;
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> event_pool;
  KStat kstat[5];                      // 0 bsp_update, 1 asp_replay, 2 local_sum, 3 scatter, 4 window with BSP events
  std::string err;
};

namespace {

ss_status fail(ss_ctx *c, ss_status s, const char *fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

// On failure the runtime's last-error slot is cleared (cudaGetLastError): a recoverable error (an allocation that
// failed) must not resurface as the launch status of a later kernel.
#define SS_CUDA(c, call)                                                                                 \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess) {                                                                             \
      cudaGetLastError();                                                                                \
      return fail((c), e_ == cudaErrorMemoryAllocation ? SS_E_OOM : SS_E_CUDA, "%s: %s (%s:%d)", #call, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                                           \
    }                                                                                                    \
  } while (0)

#define SS_NCCL(c, call)                                                                                        \
  do {                                                                                                          \
    ncclResult_t r_ = (call);                                                                                   \
    if (r_ != ncclSuccess)                                                                                      \
      return fail((c), SS_E_NCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__);         \
  } while (0)

#define SS_TRY(expr)              \
  do {                            \
    ss_status s_ = (expr);        \
    if (s_ != SS_OK) return s_;   \
  } while (0)

// Device or host memory? UVA keeps device and host virtual ranges disjoint while the context lives, so a pointer
// once seen as device memory stays device memory: remember those (the query costs ~1 us per call).
bool is_host_ptr(const void *p) {
  static thread_local std::unordered_set<const void *> device_seen;
  if (device_seen.count(p)) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  const bool host = at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
  if (!host && device_seen.size() < 4096) device_seen.insert(p);
  return host;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int32_t host_of(const ss_ctx *c, int32_t j) { return (int32_t)(((int64_t)j * c->world) / c->n); }

// lr(version, protocol) = (float)((double)eta * factor(version) * scale(protocol)) — P:1600.
float lr_at(const ss_ctx *c, int64_t ver, int32_t proto) {
  double f = 1.0;
  for (size_t i = 0; i < c->bounds.size(); ++i)
    if (c->bounds[i] <= ver) f = (double)c->factors[i];
  double scale;
  if (proto == SS_BSP) scale = (double)c->n_members;   // linear scaling over the BSP workers
  else if (c->asp_rule == 0) scale = 1.0 / std::sqrt((double)c->n);
  else if (c->asp_rule == 1) scale = 1.0 / (double)c->n;
  else scale = 1.0;
  return (float)((double)c->eta * f * scale);
}

// Momentum of an ASP push (P:1458 / P:618-619): (i) 0, (ii) 1/n, (iii) 2^i/n, (iv) i/n with i = completed epochs since
// the switch to ASP (each push is B samples); ramps stop at the BSP value; rule 0 keeps the BSP momentum.
float asp_momentum(const ss_ctx *c, int64_t ver) {
  if (c->mom_rule == 0) return c->mu;
  const int64_t i = (ver - c->asp_since) * c->mom_batch / c->mom_epoch_samples;
  double m;
  if (c->mom_rule == 1) m = 0.0;
  else if (c->mom_rule == 2) m = 1.0 / (double)c->n;
  else if (c->mom_rule == 3) m = std::ldexp(1.0, (int)std::min<int64_t>(i, 1000)) / (double)c->n;
  else m = (double)i / (double)c->n;
  return (float)std::min(m, (double)c->mu);
}

void record(ss_ctx *c, int64_t worker, int64_t b, int64_t st) {
  if ((size_t)st >= c->hist.size()) c->hist.resize((size_t)st + 1, 0);
  c->hist[st] += 1;
  c->log.push_back(worker);
  c->log.push_back(b);
  c->log.push_back(st);
  c->log.push_back(c->version);
}

// Staging slots form a ring: the pool grows to stage_cap() slots, then the oldest slot is reused. A slot taken for an
// H2D waits (on copy_in) for its previous user to be done with it, a slot a kernel will write (host pull) makes the
// compute stream wait the same way, so reuse is always ordered; the ring keeps consecutive windows on distinct slots
// when memory allows, so the waits rarely stall. Slots are taken after any window cut (enqueue), so the slots of one
// window or superstep are distinct as long as the pool holds max(n, window) of them.
int32_t stage_cap(const ss_ctx *c) {
  const int64_t need = std::max<int64_t>(c->n, c->max_win);
  const int64_t slot_bytes = std::max<int64_t>(1, c->P_pad * (int64_t)sizeof(float));
  const int64_t budget = (int64_t)24 << 30;   // prefer a whole step's worth (BSP gradients + ASP pushes and pulls)
  return (int32_t)std::max<int64_t>(need, std::min<int64_t>(4 * need, budget / slot_bytes));
}

ss_status stage_slot(ss_ctx *c, float **out, int32_t *index, bool kernel_writes) {
  if (c->capturing) return fail(c, SS_E_STATE, "host buffers cannot be used while capturing a graph");
  int32_t i;
  if ((int32_t)c->stage.size() < stage_cap(c)) {
    float *p = nullptr;
    cudaEvent_t f, r;
    SS_CUDA(c, cudaMalloc(&p, (size_t)c->P_pad * sizeof(float)));
    SS_CUDA(c, cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
    SS_CUDA(c, cudaEventCreateWithFlags(&r, cudaEventDisableTiming));
    c->stage.push_back(p);
    c->slot_free.push_back(f);
    c->slot_ready.push_back(r);
    c->slot_armed.push_back(0);
    i = (int32_t)c->stage.size() - 1;
  } else {
    i = c->stage_next;
    c->stage_next = (i + 1) % (int32_t)c->stage.size();
  }
  if (kernel_writes && c->slot_armed[i]) SS_CUDA(c, cudaStreamWaitEvent(c->stream, c->slot_free[i], 0));
  c->win_slots.push_back(i);
  if (index) *index = i;
  *out = c->stage[i];
  return SS_OK;
}

bool split_copies(const ss_ctx *c) { return c->copy_in != nullptr; }

// Host gradient -> device staging slot (the caller's buffer is borrowed until ss_sync). The H2D runs on copy_in after
// the slot's previous user is done with it, and the compute stream waits only for this copy.
ss_status resolve_src(ss_ctx *c, const float *g, const float **out) {
  if (!is_host_ptr(g)) {
    *out = g;
    return SS_OK;
  }
  float *slot = nullptr;
  int32_t i = 0;
  SS_TRY(stage_slot(c, &slot, &i, false));
  if (split_copies(c)) {
    if (c->slot_armed[i]) SS_CUDA(c, cudaStreamWaitEvent(c->copy_in, c->slot_free[i], 0));
    SS_CUDA(c, cudaMemcpyAsync(slot, g, (size_t)c->P * sizeof(float), cudaMemcpyHostToDevice, c->copy_in));
    SS_CUDA(c, cudaEventRecord(c->slot_ready[i], c->copy_in));
    SS_CUDA(c, cudaStreamWaitEvent(c->stream, c->slot_ready[i], 0));
  } else {
    SS_CUDA(c, cudaMemcpyAsync(slot, g, (size_t)c->P * sizeof(float), cudaMemcpyHostToDevice, c->stream));
  }
  *out = slot;
  return SS_OK;
}

// After the kernels that read the window's / superstep's slots were enqueued: gradient slots may be refilled once
// they are done; a host pull's slot is released by its D2H (pull_to_host).
ss_status release_slots(ss_ctx *c, const std::vector<Ev> *win = nullptr) {
  if (split_copies(c))
    for (int32_t i : c->win_slots) {
      bool pull = false;
      if (win)
        for (const Ev &e : *win) pull = pull || (e.kind == 1 && e.host_dst && e.slot == i);
      if (pull) continue;
      SS_CUDA(c, cudaEventRecord(c->slot_free[i], c->stream));
      c->slot_armed[i] = 1;
    }
  c->win_slots.clear();
  return SS_OK;
}

// A pull into host memory: D2H from its staging slot on copy_out once the window's kernel wrote it; the slot is free
// again when the copy is done.
ss_status pull_to_host(ss_ctx *c, const Ev &e) {
  if (!split_copies(c) || e.slot < 0) {
    SS_CUDA(c, cudaMemcpyAsync(e.host_dst, e.dst, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    return SS_OK;
  }
  SS_CUDA(c, cudaEventRecord(c->slot_ready[e.slot], c->stream));
  SS_CUDA(c, cudaStreamWaitEvent(c->copy_out, c->slot_ready[e.slot], 0));
  SS_CUDA(c, cudaMemcpyAsync(e.host_dst, e.dst, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToHost, c->copy_out));
  SS_CUDA(c, cudaEventRecord(c->slot_free[e.slot], c->copy_out));
  c->slot_armed[e.slot] = 1;
  return SS_OK;
}

cudaEvent_t pooled_event(ss_ctx *c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void timed_begin(ss_ctx *c, Timed *t, int kernel, double bytes, double nvbytes = 0.0) {
  if (!c->prof) return;
  t->kernel = kernel;
  t->bytes = bytes;
  t->nvbytes = nvbytes;
  t->a = pooled_event(c);
  t->b = pooled_event(c);
  cudaEventRecord(t->a, c->stream);
}

void timed_end(ss_ctx *c, Timed *t) {
  if (!c->prof) return;
  cudaEventRecord(t->b, c->stream);
  c->timed.push_back(*t);
}

ss_status drain_timed(ss_ctx *c) {
  if (c->timed.empty()) return SS_OK;
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  for (auto &t : c->timed) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    c->kstat[t.kernel].launches += 1;
    c->kstat[t.kernel].ms += ms;
    c->kstat[t.kernel].bytes += t.bytes;
    c->kstat[t.kernel].nvbytes += t.nvbytes;
    c->event_pool.push_back(t.a);
    c->event_pool.push_back(t.b);
  }
  c->timed.clear();
  return SS_OK;
}

ss_status ensure_dist_buffers(ss_ctx *c) {
  if (c->world == 1) return SS_OK;
  if (!c->sum_buf) SS_CUDA(c, cudaMalloc(&c->sum_buf, (size_t)c->P_pad * sizeof(float)));
  if (!c->rs_buf) SS_CUDA(c, cudaMalloc(&c->rs_buf, (size_t)c->reg_len * sizeof(float)));
  while ((int32_t)c->rslot.size() < c->max_win) {
    float *a = nullptr, *b = nullptr;
    SS_CUDA(c, cudaMalloc(&a, (size_t)c->reg_len * sizeof(float)));
    SS_CUDA(c, cudaMalloc(&b, (size_t)c->reg_len * sizeof(float)));
    c->rslot.push_back(a);
    c->sslot.push_back(b);
  }
  return SS_OK;
}

// ---------------------------------------------------------------------------------------------------------------
// Fused peer-memory path setup (collective): allocate the inbox / pull buffers / flag block, exchange CUDA IPC
// handles with one NCCL all-gather, map every peer's buffers. Re-run when more inbox slots are needed.
// Unmaps the peers and frees the inbox; `all` also frees the pull buffers and the flag block (destroy only: they
// keep their addresses — ss_pull_buffer hands them out — and the flags keep their epochs across re-setups).
void close_ipc(ss_ctx *c, bool all) {
  for (void *p : c->opened) cudaIpcCloseMemHandle(p);
  c->opened.clear();
  cudaFree(c->inbox);
  c->inbox = nullptr;
  c->ipc_ready = false;
  if (all) {
    cudaFree(c->pbuf);
    cudaFree(c->gbuf);
    cudaFree(c->sigblk);
    c->pbuf = nullptr;
    c->gbuf = nullptr;
    c->sigblk = nullptr;
  }
}

// NVLS replica (collective, once): every rank checks support, all agree (NCCL min), then the multicast object is
// created, shared and bound (nvls.cpp) and w moves into it. Any failure on any rank leaves every rank on the P2P
// broadcast.
ss_status agree_all(ss_ctx *c, int32_t *flag) {
  int32_t *d = nullptr;
  SS_CUDA(c, cudaMalloc(&d, sizeof(int32_t)));
  SS_CUDA(c, cudaMemcpy(d, flag, sizeof(int32_t), cudaMemcpyHostToDevice));
  SS_NCCL(c, ncclAllReduce(d, d, 1, ncclInt32, ncclMin, c->comm, c->stream));
  SS_CUDA(c, cudaMemcpyAsync(flag, d, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(d);
  return SS_OK;
}

ss_status ensure_nvls(ss_ctx *c) {
  if (c->nvls_tried) return SS_OK;
  c->nvls_tried = true;
  // Opt-in (SS_NVLS=1), off by default at every world size. Measured on this pool: at 4 GPUs a multicast store
  // moves 181 GB/s of source data per GPU against 225 GB/s for P2P stores to all three peers
  // (profiles/r01_nvls_microbench.txt), and the whole owner exchange — multimem.ld_reduce + multimem.st against P2P
  // loads + P2P stores — reaches 76% vs 75% of 900 GB/s bus bandwidth at 4 GPUs and 40% vs 65% at 2
  // (tools/nvls_reduce_bench.cu, profiles/r02_nvls_reduce_microbench.txt): no gain measured anywhere, so every world
  // size runs the P2P code the 2- and 4-GPU tests cover.
  const char *env = getenv("SS_NVLS");
  const bool want = env && env[0] == '1';
  int32_t ok = want && ss::nvls_supported(c->device) ? 1 : 0;
  SS_TRY(agree_all(c, &ok));
  if (!ok) return SS_OK;
  const char *why = ss::nvls_share(&c->nvls, c->rank, c->world, c->device, (size_t)c->P_pad * sizeof(float),
                                   c->job_tag);
  ok = why == nullptr;
  SS_TRY(agree_all(c, &ok));   // binding blocks until every rank added its device: bind only if all of them did
  if (ok) {
    why = ss::nvls_bind(&c->nvls);
    ok = why == nullptr;
    SS_TRY(agree_all(c, &ok));
  }
  if (!ok) {
    if (why) fprintf(stderr, "syncswitch: NVLS multicast unavailable on rank %d (%s); using P2P stores\n", c->rank,
                     why);
    ss::nvls_release(&c->nvls);
    return SS_OK;
  }
  SS_CUDA(c, cudaMemcpyAsync(c->nvls.uc, c->w, (size_t)c->P_pad * sizeof(float), cudaMemcpyDeviceToDevice,
                             c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(c->w);
  c->w = (float *)c->nvls.uc;
  c->w_vmm = true;
  return SS_OK;
}

ss_status ensure_fused(ss_ctx *c, int64_t slots) {
  if (c->ipc_ready && c->inbox_slots >= slots) return SS_OK;
  if (c->world > ss::kMaxPeers) return fail(c, SS_E_INVAL, "fused path supports at most %d ranks", ss::kMaxPeers);
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  close_ipc(c, false);
  slots = std::max<int64_t>(slots, std::max<int64_t>(c->n, c->max_win));
  // Two inbox buffers when every rank can afford them: consecutive exchanges then write different buffers, so a
  // rank's next phase A can never overwrite slices a peer's phase B is still reading, and the phase-B kernels need no
  // end barrier (see end_wait_needed). Any rank short of memory keeps all ranks on one buffer and end barriers.
  int32_t two = getenv("SS_INBOX_BUFS") && getenv("SS_INBOX_BUFS")[0] == '1' ? 0 : 1;
  if (two && cudaMalloc(&c->inbox, 2 * (size_t)slots * c->reg_len * sizeof(float)) != cudaSuccess) {
    cudaGetLastError();
    c->inbox = nullptr;
    two = 0;
  }
  SS_TRY(agree_all(c, &two));
  if (!two) {
    cudaFree(c->inbox);
    SS_CUDA(c, cudaMalloc(&c->inbox, (size_t)slots * c->reg_len * sizeof(float)));
  }
  c->inbox_bufs = two ? 2 : 1;
  if (!c->pbuf) SS_CUDA(c, cudaMalloc(&c->pbuf, (size_t)std::max(c->n_hosted, 1) * c->P_pad * sizeof(float)));
  if (!c->gbuf) {   // gradient buffers (mode 3): the padding stays zero, like every padded vector
    SS_CUDA(c, cudaMalloc(&c->gbuf, (size_t)std::max(c->n_hosted, 1) * c->P_pad * sizeof(float)));
    SS_CUDA(c, cudaMemset(c->gbuf, 0, (size_t)std::max(c->n_hosted, 1) * c->P_pad * sizeof(float)));
  }
  if (!c->trace_dev && getenv("SS_TRACE") && getenv("SS_TRACE")[0]) {
    c->trace_path = getenv("SS_TRACE");
    const char *cap = getenv("SS_TRACE_CAP");
    c->trace_cap = cap ? std::max<int64_t>(1, atoll(cap)) : 65536;
    SS_CUDA(c, cudaMalloc(&c->trace_dev, (size_t)c->trace_cap * 4 * sizeof(unsigned long long)));
    SS_CUDA(c, cudaMemset(c->trace_dev, 0, (size_t)c->trace_cap * 4 * sizeof(unsigned long long)));
  }
  if (!c->sigblk) {
    SS_CUDA(c, cudaMalloc(&c->sigblk, ss::kSigWords * sizeof(uint32_t)));
    SS_CUDA(c, cudaMemset(c->sigblk, 0, ss::kSigWords * sizeof(uint32_t)));
  }
  c->inbox_slots = slots;
  SS_TRY(ensure_nvls(c));
  constexpr int kH = 5;   // exported buffers: w, inbox, pull buffers, flag block, gradient buffers
  cudaIpcMemHandle_t mine[kH];
  std::memset(mine, 0, sizeof mine);
  if (!c->w_vmm) SS_CUDA(c, cudaIpcGetMemHandle(&mine[0], c->w));  // an NVLS replica is reached by multicast
  SS_CUDA(c, cudaIpcGetMemHandle(&mine[1], c->inbox));
  SS_CUDA(c, cudaIpcGetMemHandle(&mine[2], c->pbuf));
  SS_CUDA(c, cudaIpcGetMemHandle(&mine[3], c->sigblk));
  SS_CUDA(c, cudaIpcGetMemHandle(&mine[4], c->gbuf));
  char *dev = nullptr;
  const size_t per = sizeof mine;
  SS_CUDA(c, cudaMalloc(&dev, per * c->world));
  SS_CUDA(c, cudaMemcpy(dev + per * c->rank, mine, per, cudaMemcpyHostToDevice));
  SS_NCCL(c, ncclAllGather(dev + per * c->rank, dev, per, ncclChar, c->comm, c->stream));
  std::vector<cudaIpcMemHandle_t> all(kH * c->world);
  SS_CUDA(c, cudaMemcpyAsync(all.data(), dev, per * c->world, cudaMemcpyDeviceToHost, c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(dev);
  for (int32_t q = 0; q < c->world; ++q) {
    if (q == c->rank) {
      c->peer_w[q] = c->w;
      c->peer_inbox[q] = c->inbox;
      c->peer_pbuf[q] = c->pbuf;
      c->peer_sig[q] = c->sigblk;
      c->peer_gbuf[q] = c->gbuf;
      continue;
    }
    void *p[kH] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    for (int k = c->w_vmm ? 1 : 0; k < kH; ++k) {
      SS_CUDA(c, cudaIpcOpenMemHandle(&p[k], all[kH * q + k], cudaIpcMemLazyEnablePeerAccess));
      c->opened.push_back(p[k]);
    }
    c->peer_w[q] = (float *)p[0];
    c->peer_inbox[q] = (float *)p[1];
    c->peer_pbuf[q] = (float *)p[2];
    c->peer_sig[q] = (uint32_t *)p[3];
    c->peer_gbuf[q] = (float *)p[4];
  }
  // every rank has mapped every peer before anyone signals through the mappings
  SS_NCCL(c, ncclAllGather(c->sigblk + 128 + c->rank, c->sigblk + 128, 1, ncclUint32, c->comm, c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  c->ipc_ready = true;
  return SS_OK;
}

constexpr int kSigEpochBase = 160;   // sigblk word: this rank's epoch counter, advanced by the fused kernels

ss::PeerSync peer_sync(ss_ctx *c, uint32_t wait_epoch, uint32_t signal_epoch, bool end_wait, int kind) {
  ss::PeerSync p;
  std::memset(&p, 0, sizeof p);
  if (c->trace_dev && (int64_t)c->trace_kind.size() < c->trace_cap) {
    p.trace = c->trace_dev + 4 * c->trace_kind.size();
    c->trace_kind.push_back((int8_t)kind);
  }
  p.sig_local = c->sigblk;
  for (int32_t q = 0; q < c->world; ++q) p.sig_peer[q] = c->peer_sig[q];
  p.ctr = c->sigblk + 32;
  p.err = reinterpret_cast<int *>(c->sigblk + 64);
  p.rank = c->rank;
  p.world = c->world;
  // epochs travel as offsets from the device-resident counter (kSigEpochBase), whose value before this launch the
  // host mirrors in dev_epoch: identical to absolute epochs eagerly, and still correct when a graph is replayed
  p.epoch_base = c->sigblk + kSigEpochBase;
  p.has_wait = wait_epoch != 0;
  p.wait_off = wait_epoch - c->dev_epoch;
  p.signal_off = signal_epoch ? signal_epoch - c->dev_epoch : 0u;
  if (signal_epoch) c->dev_epoch = signal_epoch;
  p.end_wait = end_wait ? 1 : 0;
  return p;
}

// Inbox buffer of the exchange being issued (element offset into every rank's inbox allocation).
int64_t inbox_off(const ss_ctx *c) {
  return c->inbox_bufs == 2 ? (c->xchg & 1) * c->inbox_slots * c->reg_len : 0;
}

// Does a phase-B kernel have to wait, at its end, until every rank finished its phase B? Only when something after
// it on this rank's stream depends on the peers' stores being complete (a hosted pull copied out of its pull buffer),
// or when the inbox is single-buffered (the next phase A would overwrite slices still being read). With two buffers,
// exchange x's phase A on one rank starts only after that rank's phase B of x-1 saw every rank's phase A of x-1 —
// which each rank issued after finishing its phase B of x-2, the last reader of the buffer x reuses. A captured
// graph bakes its exchanges' buffers in: an even number per capture keeps the alternation across replays, an odd
// number gets a closing barrier (ss_capture_end).
bool end_wait_needed(const ss_ctx *c, bool copy_follows) {
  return copy_follows || c->inbox_bufs == 1 || c->nvls.ready;
}

// Phase A of every fused exchange: hosted sources' owner slices -> owners' inbox slots, then signal `epoch`.
ss_status launch_scatter(ss_ctx *c, const std::vector<std::pair<const float *, int32_t>> &src, uint32_t epoch) {
  ss::ScatterArgs a;
  std::memset(&a, 0, sizeof a);
  a.n_src = (int32_t)src.size();
  for (size_t k = 0; k < src.size(); ++k) {
    a.src[k] = src[k].first;
    a.slot[k] = src[k].second;
    if (!aligned16(src[k].first)) return fail(c, SS_E_INVAL, "fused path needs 16-byte aligned gradients");
  }
  for (int32_t q = 0; q < c->world; ++q) a.inbox[q] = c->peer_inbox[q] + inbox_off(c);
  a.reg_len = c->reg_len;
  a.P = c->P;
  a.sync = peer_sync(c, 0, epoch, false, 0);
  Timed t;
  double remote = 0.0;  // elements of the other ranks' regions
  for (int32_t q = 0; q < c->world; ++q)
    if (q != c->rank) remote += (double)(c->real_hi[q] - c->real_lo[q]);
  timed_begin(c, &t, 3, 4.0 * remote * (double)src.size(), 4.0 * remote * (double)src.size());
  SS_CUDA(c, ss::launch_scatter(a, c->stream));
  timed_end(c, &t);
  return SS_OK;
}

// ---------------------------------------------------------------------------------------------------------------
// ASP window flush: [G>1: grouped send/recv of gradient shards to owners] -> asp_replay on the owned slice ->
// [G>1: grouped send/recv of snapshot shards to pullers] -> D2H of host destinations.
int32_t first_hosted_of(const ss_ctx *c, int32_t rank) {
  int32_t j = 0;
  while (j < c->n && host_of(c, j) < rank) ++j;
  return j;
}

// Fused ASP window (G > 1): scatter the hosted pushes' owner slices (phase A), then every owner replays the window on
// its slice and stores each pull's snapshot slice straight into the puller's mapped pull buffer (phase B); hosted
// pulls are then copied from the pull buffer to the caller's destination.
ss_status flush_fused(ss_ctx *c) {
  SS_TRY(ensure_fused(c, c->max_win));
  const int32_t me = c->rank;
  const int64_t lo = c->real_lo[me], cnt = c->real_hi[me] - lo;
  const uint32_t epA = ++c->epoch, epB = ++c->epoch;
  std::vector<std::pair<const float *, int32_t>> src;
  for (size_t k = 0; k < c->win.size(); ++k) {
    const Ev &e = c->win[k];
    if (e.kind == 0 && host_of(c, e.worker) == me) src.push_back({e.src, (int32_t)k});
  }
  SS_TRY(launch_scatter(c, src, epA));
  ss::AspArgs a;
  std::memset(&a, 0, sizeof a);
  bool vec = true;
  int32_t ne = 0, n_push = 0, n_pull = 0, n_remote_pull = 0;
  for (size_t k = 0; k < c->win.size(); ++k) {
    const Ev &e = c->win[k];
    if (e.kind == 1 && e.data && host_of(c, e.worker) != me) ++n_remote_pull;
    ss::AspEvent &x = a.ev[ne];
    x.kind = e.kind;
    if (e.kind == 0) {
      x.src = host_of(c, e.worker) == me ? e.src + lo : c->inbox + inbox_off(c) + (int64_t)k * c->reg_len;
      x.lr = e.lr;
      x.mu = e.mu;
      vec = vec && aligned16(x.src);
      ++n_push;
    } else {
      if (!e.data) continue;
      const int32_t h = host_of(c, e.worker);
      x.dst = c->peer_pbuf[h] + (int64_t)(e.worker - first_hosted_of(c, h)) * c->P_pad + lo;
      ++n_pull;
    }
    ++ne;
  }
  a.n_ev = ne;
  a.w = c->w + lo;
  a.v = c->v;
  a.flag = c->flag;
  a.count = cnt;
  a.lam = c->lam;
  a.nesterov = c->nesterov;
  bool copy_follows = false;
  for (const Ev &e : c->win)
    if (e.kind == 1 && e.data && host_of(c, e.worker) == me &&
        e.dst != c->pbuf + (int64_t)(e.worker - c->first_hosted) * c->P_pad)
      copy_follows = true;
  a.sync = peer_sync(c, epA, epB, end_wait_needed(c, copy_follows), 3);
  Timed t;
  timed_begin(c, &t, 1, 4.0 * (double)cnt * (4 + n_push + n_pull), 4.0 * (double)cnt * n_remote_pull);
  SS_CUDA(c, ss::launch_asp_replay(a, vec, c->stream));
  timed_end(c, &t);
  c->xchg += 1;
  // gradient slots are free once the kernels that read them are done (host pulls keep theirs until their D2H)
  SS_TRY(release_slots(c, &c->win));
  for (const Ev &e : c->win) {
    if (e.kind != 1 || !e.data || host_of(c, e.worker) != me) continue;
    const float *pb = c->pbuf + (int64_t)(e.worker - c->first_hosted) * c->P_pad;
    if (e.dst == pb) continue;  // zero-copy pull into the mapped pull buffer (ss_pull_buffer)
    // the pull buffer is rewritten by the owners in the next window, which cannot start before this rank's next
    // kernel: copy it out on the compute stream (into the staging slot for a host destination, whose D2H then runs
    // on copy_out, overlapping the next window)
    SS_CUDA(c, cudaMemcpyAsync(e.dst, pb, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
    if (e.host_dst) SS_TRY(pull_to_host(c, e));
  }
  c->win.clear();
  c->win_kind.clear();
  c->win_worker.clear();
  c->win_bsp_src.clear();
  return SS_OK;
}

ss_status flush(ss_ctx *c) {
  if (c->win.empty()) return SS_OK;
  if (c->world > 1 && c->fused_mode != 0) return flush_fused(c);
  const int32_t me = c->rank;
  const int64_t lo = c->real_lo[me], hi = c->real_hi[me], cnt = hi - lo;
  int32_t n_push = 0, n_pull = 0, n_bsp_src = 0;
  for (const Ev &e : c->win) {
    if (e.kind == 0) ++n_push;
    else if (e.kind == 2) n_bsp_src += e.n_src;
    else if (e.data) ++n_pull;
  }

  // routing plan of this window (plan.h; the same code ss_route_plan exposes to the CPU tests)
  std::vector<ss::RouteOp> plan;
  if (c->world > 1) {
    std::vector<int32_t> kd, wk;
    std::vector<uint8_t> dt;
    for (const Ev &e : c->win) {
      kd.push_back(e.kind);
      wk.push_back(e.worker);
      dt.push_back(e.data ? 1 : 0);
    }
    ss::plan_window(c->L, kd.data(), wk.data(), dt.data(), (int32_t)kd.size(), plan);
    SS_TRY(ensure_dist_buffers(c));
    SS_NCCL(c, ncclGroupStart());
    for (const ss::RouteOp &o : plan) {
      if (o.phase != 0) continue;
      if (o.op == 0)
        SS_NCCL(c, ncclSend(c->win[o.event].src + o.offset, o.count, ncclFloat, o.peer, c->comm, c->stream));
      else
        SS_NCCL(c, ncclRecv(c->rslot[o.event], o.count, ncclFloat, o.peer, c->comm, c->stream));
    }
    SS_NCCL(c, ncclGroupEnd());
  }

  if (cnt > 0) {
    // A lone superstep of a large vector runs in bsp_update (config 3: 0.977 vs 0.918 of HBM through the window
    // kernel); below 2^20 parameters the window kernel's small-launch form is the faster one (config 2: 63.7k vs
    // 61.5k steps/s eager, profiles/r02_lone_superstep_ab.txt)
    if (c->world == 1 && c->win.size() == 1 && c->win[0].kind == 2 && c->P > (int64_t)1 << 20) {
      // a lone superstep (flushed at its data dependency): the streaming aggregate-and-update kernel, which reads
      // each gradient once and w, v once — the same arithmetic as the window kernel's BSP event
      const Ev &e = c->win[0];
      ss::BspArgs a;
      std::memset(&a, 0, sizeof a);
      bool vec = aligned16(c->w) && aligned16(c->v);
      for (int32_t k = 0; k < e.n_src; ++k) {
        a.g[k] = c->win_bsp_src[e.src0 + k];
        vec = vec && aligned16(a.g[k]);
      }
      a.n_in = e.n_src;
      a.flag = c->flag;
      a.divisor = e.divisor;
      a.mu = e.mu;
      a.neg_eta = -e.lr;
      a.lam = c->lam;
      a.nesterov = c->nesterov;
      a.w = c->w;
      a.v = c->v;
      a.count = c->P;
      Timed t;
      timed_begin(c, &t, 0, 4.0 * (double)c->P * (e.n_src + 4));
      SS_CUDA(c, ss::launch_bsp_update(a, vec, c->stream));
      timed_end(c, &t);
    } else if (n_push == 0 && n_bsp_src == 0 && c->world == 1) {
      // pulls only: plain copies of the current w
      for (const Ev &e : c->win)
        if (e.data) SS_CUDA(c, cudaMemcpyAsync(e.dst, c->w, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToDevice,
                                              c->stream));
    } else {
      ss::AspArgs a;
      std::memset(&a, 0, sizeof a);
      bool vec = true;
      int32_t ne = 0;
      for (size_t k = 0; k < c->win.size(); ++k) {
        const Ev &e = c->win[k];
        ss::AspEvent &x = a.ev[ne];
        x.kind = e.kind;
        if (e.kind == 0) {
          x.src = (c->world == 1 || host_of(c, e.worker) == me) ? e.src + lo : c->rslot[k];
          x.lr = e.lr;
          x.mu = e.mu;
          vec = vec && aligned16(x.src);
        } else if (e.kind == 2) {   // one GPU only: the superstep's gradients in ascending worker order
          x.lr = e.lr;
          x.mu = e.mu;
          x.divisor = e.divisor;
          x.src0 = e.src0;
          x.n_src = e.n_src;
        } else {
          if (!e.data) continue;  // version-only pull: no data
          x.dst = (c->world == 1 || host_of(c, e.worker) == me) ? e.dst + lo : c->sslot[k];
          vec = vec && aligned16(x.dst);
        }
        ++ne;
      }
      for (size_t k = 0; k < c->win_bsp_src.size(); ++k) {
        a.bsp_src[k] = c->win_bsp_src[k];
        vec = vec && aligned16(a.bsp_src[k]);
      }
      a.n_ev = ne;
      a.w = c->w + lo;
      a.v = c->v;
      a.flag = c->flag;
      a.count = cnt;
      a.lam = c->lam;
      a.nesterov = c->nesterov;
      Timed t;
      timed_begin(c, &t, n_bsp_src ? 4 : 1, 4.0 * (double)cnt * (4 + n_push + n_pull + n_bsp_src));
      SS_CUDA(c, ss::launch_asp_replay(a, vec, c->stream));
      timed_end(c, &t);
    }
  }

  if (c->world > 1) {
    SS_NCCL(c, ncclGroupStart());
    for (const ss::RouteOp &o : plan) {
      if (o.phase != 1) continue;
      if (o.op == 0)
        SS_NCCL(c, ncclSend(c->sslot[o.event], o.count, ncclFloat, o.peer, c->comm, c->stream));
      else
        SS_NCCL(c, ncclRecv(c->win[o.event].dst + o.offset, o.count, ncclFloat, o.peer, c->comm, c->stream));
    }
    SS_NCCL(c, ncclGroupEnd());
  }

  // slots read by the kernel (gradients) are free after it; host pulls free theirs after their D2H
  SS_TRY(release_slots(c, &c->win));
  for (const Ev &e : c->win)
    if (e.kind == 1 && e.host_dst) SS_TRY(pull_to_host(c, e));
  c->win.clear();
  c->win_kind.clear();
  c->win_worker.clear();
  c->win_bsp_src.clear();
  return SS_OK;
}

// A pending switch takes effect once version >= at (SV §8c maybe_switch). ASP->BSP: pending window flushed, later
// pushes of the old phase are rejected and counted (reading C8), every worker's base version becomes V.
ss_status maybe_switch(ss_ctx *c) {
  if (c->has_pending && c->version >= c->pending_at) {
    c->has_pending = false;
    if (c->pending_proto != c->proto) {
      // one GPU: every queued event carries its own lr / momentum, so the window may span the switch; at G > 1 BSP
      // runs outside the windows (exchange kernels), so the ASP window is applied first
      if (c->world > 1) SS_TRY(flush(c));
      c->proto = c->pending_proto;
      if (c->proto == SS_BSP)
        for (auto &b : c->base) b = c->version;
      else
        c->asp_since = c->version;
    }
  }
  return SS_OK;
}

ss_status check_live(ss_ctx *c) {
  if (!c) return SS_E_INVAL;
  if (c->diverged) return fail(c, SS_E_DIVERGED, "diverged: a non-finite parameter or momentum was produced");
  return SS_OK;
}

// Appending an event to the pending window is split so that a call either applies completely or not at all (SV §8b
// "errors never partially apply"): enqueue_prepare does everything that can fail — the capture check for host
// buffers, the window cut (device work of earlier, already accepted calls), the staging of host data — before the
// caller touches any protocol state; enqueue_commit cannot fail. The event's staging follows the cut, so a window's
// slots all belong to it. win_kind / win_worker mirror the window for the cut rule (no per-call rebuild).
ss_status enqueue_prepare(ss_ctx *c, Ev &e, const float *src, float *pull_dst) {
  if (c->capturing && ((src && is_host_ptr(src)) || (pull_dst && is_host_ptr(pull_dst))))
    return fail(c, SS_E_STATE, "host buffers cannot be used while capturing a graph");
  if (ss::window_cut(c->win_kind.data(), c->win_worker.data(), (int32_t)c->win_kind.size(), e.kind, e.worker,
                     c->max_win, c->world > 1 && c->fused_mode != 0) ||
      (int32_t)c->win.size() >= ss::kMaxEvents)
    SS_TRY(flush(c));
  if (e.kind == 0 && src) SS_TRY(resolve_src(c, src, &e.src));
  if (e.kind == 1 && pull_dst) {
    if (is_host_ptr(pull_dst)) {
      float *slot = nullptr;
      SS_TRY(stage_slot(c, &slot, &e.slot, true));
      e.dst = slot;
      e.host_dst = pull_dst;
    } else {
      e.dst = pull_dst;
    }
  }
  return SS_OK;
}

void enqueue_commit(ss_ctx *c, const Ev &e) {
  c->win.push_back(e);
  if (e.kind == 2) return;
  c->win_kind.push_back(e.kind);
  c->win_worker.push_back(e.worker);
}

// A window holding max_win ASP events is launched right away (eagerly: its device work then overlaps the host's next
// calls).
ss_status flush_if_full(ss_ctx *c) { return (int32_t)c->win_kind.size() >= c->max_win ? flush(c) : SS_OK; }

// Multi-GPU: each rank's kernels see only its own owned slice, so a non-finite value or a timed-out cross-GPU
// barrier is first known to one rank. ss_sync is collective: the ranks agree on both words (NCCL max) before
// deciding, so every rank becomes DIVERGED (or reports the timeout) at the same ss_sync.
ss_status agree_health(ss_ctx *c, int *div, int *timeout) {
  if (c->world == 1 || !c->comm) return SS_OK;
  if (!c->health) SS_CUDA(c, cudaMalloc(&c->health, 2 * sizeof(int)));
  SS_CUDA(c, cudaMemcpyAsync(c->health, c->flag, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
  if (c->ipc_ready)
    SS_CUDA(c, cudaMemcpyAsync(c->health + 1, c->sigblk + 64, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
  else
    SS_CUDA(c, cudaMemsetAsync(c->health + 1, 0, sizeof(int), c->stream));
  SS_NCCL(c, ncclAllReduce(c->health, c->health, 2, ncclInt32, ncclMax, c->comm, c->stream));
  int h[2] = {0, 0};
  SS_CUDA(c, cudaMemcpyAsync(h, c->health, sizeof h, cudaMemcpyDeviceToHost, c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  *div = h[0];
  *timeout = h[1];
  return SS_OK;
}

ss_status sync_impl(ss_ctx *c) {
  SS_TRY(flush(c));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  if (c->copy_in) SS_CUDA(c, cudaStreamSynchronize(c->copy_in));
  if (c->copy_out) SS_CUDA(c, cudaStreamSynchronize(c->copy_out));
  int h = 0, t = 0;
  if (c->world > 1 && c->comm) {
    SS_TRY(agree_health(c, &h, &t));
  } else {
    SS_CUDA(c, cudaMemcpy(&h, c->flag, sizeof(int), cudaMemcpyDeviceToHost));
  }
  if (h) c->diverged = true;
  if (t) return fail(c, SS_E_CUDA, "fused path: a cross-GPU barrier timed out (a peer did not arrive)");
  if (c->diverged) return fail(c, SS_E_DIVERGED, "diverged: a non-finite parameter or momentum was produced");
  return SS_OK;
}

}  // namespace

extern "C" {

ss_status ss_init(ss_ctx **out, const float *params, int64_t n_params, int32_t n_shards, int32_t n_workers,
                  float lr, float momentum) {
  if (!out) return SS_E_INVAL;
  *out = nullptr;
  if (!params || n_params < 1 || n_shards < 1 || n_workers < 1 || n_workers > ss::kMaxWorkers || !(lr > 0.0f) ||
      !(momentum >= 0.0f && momentum < 1.0f))
    return SS_E_INVAL;
  ss_ctx *c = new (std::nothrow) ss_ctx;
  if (!c) return SS_E_OOM;
  c->P = n_params;
  c->S = n_shards;
  c->n = n_workers;
  c->eta = lr;
  c->mu = momentum;
  const int64_t per = (n_params + n_shards - 1) / n_shards;
  c->pad = ((per + 31) / 32) * 32;
  c->P_pad = c->pad * n_shards;
  c->off.resize(n_shards + 1);
  for (int32_t s = 0; s <= n_shards; ++s) c->off[s] = std::min<int64_t>((int64_t)s * c->pad, n_params);
  c->base.assign(n_workers, 0);
  c->member.assign(n_workers, 1);
  c->n_members = n_workers;
  c->L = ss::make_layout(n_params, n_shards, n_workers, 0, 1);
  c->reg_len = c->L.reg_len;
  c->real_lo = c->L.real_lo;
  c->real_hi = c->L.real_hi;
  auto bail = [&](ss_status s) {
    ss_destroy(c);
    return s;
  };
  if (cudaGetDevice(&c->device) != cudaSuccess) return bail(SS_E_CUDA);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(SS_E_CUDA);
  if (cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking) != cudaSuccess)
    return bail(SS_E_CUDA);
  if (cudaMalloc(&c->w, (size_t)c->P_pad * sizeof(float)) != cudaSuccess) return bail(SS_E_OOM);
  if (cudaMalloc(&c->v, (size_t)c->P_pad * sizeof(float)) != cudaSuccess) return bail(SS_E_OOM);
  if (cudaMalloc(&c->flag, sizeof(int)) != cudaSuccess) return bail(SS_E_OOM);
  if (cudaMemsetAsync(c->w, 0, (size_t)c->P_pad * sizeof(float), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->v, 0, (size_t)c->P_pad * sizeof(float), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->flag, 0, sizeof(int), c->stream) != cudaSuccess ||
      cudaMemcpyAsync(c->w, params, (size_t)n_params * sizeof(float), cudaMemcpyDefault, c->stream) != cudaSuccess ||
      cudaStreamSynchronize(c->stream) != cudaSuccess)
    return bail(SS_E_CUDA);
  *out = c;
  return SS_OK;
}

ss_status ss_nccl_unique_id(void *out128) {
  if (!out128) return SS_E_INVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SS_E_NCCL;
  std::memcpy(out128, &id, sizeof id);
  return SS_OK;
}

ss_status ss_init_dist(ss_ctx *c, int32_t rank, int32_t world, const void *uid) {
  SS_TRY(check_live(c));
  if (!uid || world < 1 || rank < 0 || rank >= world) return fail(c, SS_E_INVAL, "bad rank/world");
  if (c->S % world) return fail(c, SS_E_INVAL, "n_shards (%d) must be a multiple of world (%d)", c->S, world);
  if (c->stepped || c->comm) return fail(c, SS_E_STATE, "ss_init_dist must precede the first step, once");
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof id);
  SS_NCCL(c, ncclCommInitRank(&c->comm, world, id, rank));
  uint64_t h = 1469598103934665603ull;  // FNV-1a of the unique id: the same tag on every rank of this job
  for (size_t i = 0; i < sizeof id; ++i) h = (h ^ (uint8_t)id.internal[i]) * 1099511628211ull;
  std::snprintf(c->job_tag, sizeof c->job_tag, "%016llx", (unsigned long long)h);
  c->rank = rank;
  c->world = world;
  c->L = ss::make_layout(c->P, c->S, c->n, rank, world);
  c->reg_len = c->L.reg_len;
  c->real_lo = c->L.real_lo;
  c->real_hi = c->L.real_hi;
  c->first_hosted = c->L.first_hosted(rank);
  c->n_hosted = c->L.n_hosted(rank);
  // momentum now covers the owned region only
  float *v = nullptr;
  SS_CUDA(c, cudaMalloc(&v, (size_t)c->reg_len * sizeof(float)));
  SS_CUDA(c, cudaMemsetAsync(v, 0, (size_t)c->reg_len * sizeof(float), c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  cudaFree(c->v);
  c->v = v;
  return SS_OK;
}

void ss_destroy(ss_ctx *c) {
  if (!c) return;
  if (c->stream) {
    flush(c);
    cudaStreamSynchronize(c->stream);
  }
  if (c->trace_dev) {   // SS_TRACE dump: <prefix>.rank<r>.csv, one row per fused launch
    std::vector<unsigned long long> h(4 * c->trace_kind.size());
    if (!h.empty() &&
        cudaMemcpy(h.data(), c->trace_dev, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
            cudaSuccess) {
      const std::string path = c->trace_path + ".rank" + std::to_string(c->rank) + ".csv";
      if (FILE *f = fopen(path.c_str(), "w")) {
        static const char *names[] = {"scatter", "scatter_sum", "bsp_update", "asp_replay"};
        fprintf(f, "launch,kernel,enter_ns,waited_ns,signal_ns,end_ns\n");
        for (size_t i = 0; i < c->trace_kind.size(); ++i)
          fprintf(f, "%zu,%s,%llu,%llu,%llu,%llu\n", i, names[c->trace_kind[i]], h[4 * i], h[4 * i + 1],
                  h[4 * i + 2], h[4 * i + 3]);
        fclose(f);
      }
    }
    cudaFree(c->trace_dev);
  }
  for (auto &t : c->timed) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  close_ipc(c, true);
  if (c->w_vmm) {
    c->w = nullptr;            // lives in the NVLS replica
    ss::nvls_release(&c->nvls);
  }
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->copy_in) cudaStreamSynchronize(c->copy_in);
  if (c->copy_out) cudaStreamSynchronize(c->copy_out);
  for (float *p : c->stage) cudaFree(p);
  for (cudaEvent_t e : c->slot_free) cudaEventDestroy(e);
  for (cudaEvent_t e : c->slot_ready) cudaEventDestroy(e);
  if (c->copy_in) cudaStreamDestroy(c->copy_in);
  if (c->copy_out) cudaStreamDestroy(c->copy_out);
  for (float *p : c->rslot) cudaFree(p);
  for (float *p : c->sslot) cudaFree(p);
  cudaFree(c->sum_buf);
  cudaFree(c->rs_buf);
  cudaFree(c->w);
  cudaFree(c->v);
  cudaFree(c->flag);
  cudaFree(c->health);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char *ss_last_error(const ss_ctx *c) { return c ? c->err.c_str() : "null context"; }

ss_status ss_set_lr_schedule(ss_ctx *c, const int64_t *b, const float *f, int32_t nb) {
  SS_TRY(check_live(c));
  if (nb < 0 || nb > kMaxSchedule || (nb > 0 && (!b || !f))) return fail(c, SS_E_INVAL, "bad schedule");
  for (int32_t i = 0; i < nb; ++i)
    if (b[i] < 0 || !(f[i] > 0.0f) || (i > 0 && b[i] <= b[i - 1])) return fail(c, SS_E_INVAL, "bad schedule");
  c->bounds.assign(b, b + nb);
  c->factors.assign(f, f + nb);
  return SS_OK;
}

ss_status ss_set_lr_policy(ss_ctx *c, int32_t asp_rule, float weight_decay) {
  SS_TRY(check_live(c));
  if (asp_rule < 0 || asp_rule > 2 || !(weight_decay >= 0.0f)) return fail(c, SS_E_INVAL, "bad lr policy");
  SS_TRY(flush(c));  // queued pushes keep the lambda they were issued under
  c->asp_rule = asp_rule;
  c->lam = weight_decay;
  return SS_OK;
}

ss_status ss_set_nesterov(ss_ctx *c, int32_t on) {
  SS_TRY(check_live(c));
  if (on != 0 && on != 1) return fail(c, SS_E_INVAL, "nesterov must be 0 or 1");
  SS_TRY(flush(c));  // queued pushes are applied under the setting they were issued under
  c->nesterov = on;
  return SS_OK;
}

ss_status ss_set_momentum_policy(ss_ctx *c, int32_t rule, int64_t samples_per_epoch, int64_t batch) {
  SS_TRY(check_live(c));
  if (rule < 0 || rule > 4 || samples_per_epoch < 1 || batch < 1) return fail(c, SS_E_INVAL, "bad momentum policy");
  c->mom_rule = rule;
  c->mom_epoch_samples = samples_per_epoch;
  c->mom_batch = batch;
  return SS_OK;
}

ss_status ss_set_members(ss_ctx *c, const int32_t *workers, int32_t count) {
  SS_TRY(check_live(c));
  if (count < 1 || count > c->n || !workers) return fail(c, SS_E_INVAL, "member set must hold 1..n workers");
  std::vector<uint8_t> m(c->n, 0);
  for (int32_t i = 0; i < count; ++i) {
    if (workers[i] < 0 || workers[i] >= c->n || m[workers[i]])
      return fail(c, SS_E_INVAL, "bad or duplicate member %d", workers[i]);
    m[workers[i]] = 1;
  }
  c->member = m;
  c->n_members = count;
  return SS_OK;
}

ss_status ss_current_lr(ss_ctx *c, int32_t proto, float *lr_out) {
  if (!c || !lr_out || (proto != SS_BSP && proto != SS_ASP)) return SS_E_INVAL;
  *lr_out = lr_at(c, c->version, proto);
  return SS_OK;
}

ss_status ss_bsp_step(ss_ctx *c, const float *const *grads, const int32_t *workers, const int64_t *versions,
                      int32_t n_local) {
  SS_TRY(check_live(c));
  if (!grads || !workers || !versions || n_local < 0) return fail(c, SS_E_INVAL, "null argument");
  SS_TRY(maybe_switch(c));
  if (c->proto != SS_BSP) return fail(c, SS_E_STATE, "ss_bsp_step under ASP");
  // barrier: exactly the expected workers (the BSP members; multi-GPU: this rank's hosted members), each once
  // (elastic policy S:246-254)
  std::vector<const float *> by(c->n, nullptr);
  int32_t expected = 0;
  for (int32_t j = 0; j < c->n; ++j) expected += host_of(c, j) == c->rank && c->member[j];
  for (int32_t i = 0; i < n_local; ++i) {
    const int32_t j = workers[i];
    if (j < 0 || j >= c->n) return fail(c, SS_E_INVAL, "worker %d out of range", j);
    if (host_of(c, j) != c->rank) return fail(c, SS_E_PROTOCOL, "worker %d is not hosted on rank %d", j, c->rank);
    if (!c->member[j]) return fail(c, SS_E_PROTOCOL, "worker %d is not a BSP member", j);
    if (by[j] || !grads[i]) return fail(c, SS_E_PROTOCOL, "duplicate or null gradient for worker %d", j);
    by[j] = grads[i];
  }
  if (n_local != expected) return fail(c, SS_E_PROTOCOL, "missing worker: %d of %d gradients", n_local, expected);
  for (int32_t i = 0; i < n_local; ++i)
    if (versions[i] != c->version)
      return fail(c, SS_E_BARRIER, "worker %d base version %lld != current %lld", workers[i],
                  (long long)versions[i], (long long)c->version);
  if (c->world > 1 && c->fused_mode != 0)   // checked before any state changes (host buffers are staged aligned)
    for (int32_t i = 0; i < n_local; ++i)
      if (!aligned16(grads[i]) && !is_host_ptr(grads[i]))
        return fail(c, SS_E_INVAL, "fused path needs 16-byte aligned gradients");
  if (c->capturing)
    for (int32_t i = 0; i < n_local; ++i)
      if (is_host_ptr(grads[i])) return fail(c, SS_E_STATE, "host buffers cannot be used while capturing a graph");
  if (c->world == 1 && n_local <= ss::kMaxBspSrc) {
    // One GPU: the superstep joins the pending window as a BSP event (the window kernel sums its gradients in
    // ascending worker order and applies the mean and the momentum update tile by tile, with w and v on chip, before
    // the window's later pushes and pulls: bit-identical to a separate update, without the w, v round trip through
    // HBM). Room first: the window's gradient list, its event array and the staging ring must take the superstep.
    int32_t host_grads = 0;
    for (int32_t i = 0; i < n_local; ++i) host_grads += is_host_ptr(grads[i]) ? 1 : 0;
    if ((int64_t)c->win_bsp_src.size() + n_local > ss::kMaxBspSrc || (int32_t)c->win.size() >= ss::kMaxEvents ||
        (host_grads && (int64_t)c->win_slots.size() + host_grads > stage_cap(c)))
      SS_TRY(flush(c));
    Ev e{};
    e.kind = 2;
    e.lr = lr_at(c, c->version, SS_BSP);     // pre-increment version (reading C9)
    e.mu = c->mu;
    e.divisor = (float)c->n_members;
    e.src0 = (int32_t)c->win_bsp_src.size();
    std::vector<const float *> src;
    for (int32_t j = 0; j < c->n; ++j) {     // ascending worker order (reading C12)
      if (!by[j]) continue;
      const float *g = nullptr;
      SS_TRY(resolve_src(c, by[j], &g));       // may fail: nothing of this superstep is applied yet
      src.push_back(g);
    }
    e.n_src = (int32_t)src.size();
    c->win_bsp_src.insert(c->win_bsp_src.end(), src.begin(), src.end());
    enqueue_commit(c, e);
    c->stepped = true;
    for (int32_t j = 0; j < c->n; ++j)
      if (c->member[j]) record(c, j, c->version, 0);  // one staleness-0 record per BSP member
    c->version += 1;
    for (auto &b : c->base) b = c->version;
    return SS_OK;
  }
  SS_TRY(flush(c));
  c->stepped = true;

  ss::BspArgs a;
  std::memset(&a, 0, sizeof a);
  bool vec = true;
  int32_t k = 0;
  std::vector<int32_t> ids;             // hosted members, ascending
  const bool pull_mode = c->world > 1 && c->fused_mode == 3;
  for (int32_t j = 0; j < c->n; ++j) {  // ascending worker order (reading C12)
    if (!by[j]) continue;
    ids.push_back(j);
    const float *g = by[j];
    if (!pull_mode) SS_TRY(resolve_src(c, by[j], &g));   // (mode 3 copies straight into its gradient buffers)
    a.g[k++] = g;
    vec = vec && aligned16(g);
  }
  const float eta_t = lr_at(c, c->version, SS_BSP);  // pre-increment version (reading C9)
  a.flag = c->flag;
  a.divisor = (float)c->n_members;
  a.mu = c->mu;
  a.neg_eta = -eta_t;
  a.lam = c->lam;
  a.nesterov = c->nesterov;
  if (c->world == 1) {
    a.n_in = k;
    a.w = c->w;
    a.v = c->v;
    a.count = c->P;
    Timed t;
    timed_begin(c, &t, 0, 4.0 * (double)c->P * (k + 4));
    SS_CUDA(c, ss::launch_bsp_update(a, vec, c->stream));
    timed_end(c, &t);
  } else if (pull_mode) {
    // Fused pull exchange (SURVEY §8(f) NEXT-1 as one kernel, "push the computed gradients to all PSs"): every
    // rank's hosted gradients sit in its exported gradient buffers (ss_grad_buffer hands them out: zero copy; any other
    // buffer is copied in on the stream first). Each owner loads the members' slices of its region — hosted ones from
    // local HBM, the others from the peers' buffers over NVLink — sums them in ascending worker order (bit-identical to
    // one GPU), updates w and v, and stores the new slice into every replica. Cross-GPU barriers: at entry (every rank
    // signals that its gradients are in place, then waits for all) and at exit (no rank reuses a gradient buffer or
    // reads its replica before every owner is done).
    SS_TRY(ensure_fused(c, c->max_win));
    const int32_t me = c->rank;
    const int64_t lo = c->real_lo[me], cnt = c->real_hi[me] - lo;
    for (int32_t i = 0; i < k; ++i) {
      float *dst = c->gbuf + (int64_t)(ids[i] - c->first_hosted) * c->P_pad;
      if (a.g[i] != dst)
        SS_CUDA(c, cudaMemcpyAsync(dst, a.g[i], (size_t)c->P * sizeof(float), cudaMemcpyDefault, c->stream));
    }
    std::memset(a.g, 0, sizeof a.g);
    int32_t ni = 0, remote = 0;
    for (int32_t j = 0; j < c->n; ++j) {   // the members' slices, ascending worker order
      if (!c->member[j]) continue;
      const int32_t h = host_of(c, j);
      a.g[ni++] = c->peer_gbuf[h] + (int64_t)(j - first_hosted_of(c, h)) * c->P_pad + lo;
      remote += h != me;
    }
    a.n_in = ni;
    a.w = c->w + lo;
    a.v = c->v;
    a.count = cnt;
    a.n_bcast = 0;
    if (c->nvls.ready) {
      a.mc_w = (float *)c->nvls.mcv + lo;
    } else {
      for (int32_t step = 1; step < c->world; ++step)   // rotated: the ranks' stores go to distinct receivers
        a.bcast[a.n_bcast++] = c->peer_w[(me + step) % c->world] + lo;
    }
    const uint32_t epA = ++c->epoch, epB = ++c->epoch;
    a.sync = peer_sync(c, epA, epB, true, 2);
    a.sync.entry_signal = 1;
    Timed t;
    // NVLink bytes per direction: the remote slices this owner loads (the peers load as many of this rank's
    // gradients) plus the slices it stores into the other replicas (as many arrive from the other owners)
    timed_begin(c, &t, 0, 4.0 * (double)cnt * (ni + 4), 4.0 * (double)cnt * (remote + (c->world - 1)));
    if (!c->nvls.ready && ni <= ss::kMaxBspSrc) {
      // the window kernel's form (measured 0.717 vs 0.689 of 900 GB/s bus bandwidth for the register form at 4 GPUs,
      // config 5a): one BSP event whose sources — the local and peer gradient slices — are staged by 1-D bulk copies
      // (the TMA engine reads the peers' memory over NVLink), then one store event per peer replica
      ss::AspArgs r;
      std::memset(&r, 0, sizeof r);
      ss::AspEvent &x = r.ev[0];
      x.kind = 2;
      x.lr = -a.neg_eta;
      x.mu = a.mu;
      x.divisor = a.divisor;
      x.src0 = 0;
      x.n_src = ni;
      for (int32_t i = 0; i < ni; ++i) r.bsp_src[i] = a.g[i];
      for (int32_t b = 0; b < a.n_bcast; ++b) {
        r.ev[1 + b].kind = 1;
        r.ev[1 + b].dst = a.bcast[b];
      }
      r.n_ev = 1 + a.n_bcast;
      r.w = a.w;
      r.v = a.v;
      r.flag = a.flag;
      r.count = cnt;
      r.lam = a.lam;
      r.nesterov = a.nesterov;
      r.sync = a.sync;
      SS_CUDA(c, ss::launch_asp_replay(r, true, c->stream));
    } else {
      SS_CUDA(c, ss::launch_bsp_update(a, true, c->stream));   // NVLS (opt-in) multicast stores; > 128 members
    }
    timed_end(c, &t);
    c->xchg += 1;
  } else if (c->fused_mode != 0) {
    // Fused peer-memory BSP. Phase A: scatter hosted gradients (exact mode) or this rank's
    // pre-sum (mode 2) into the owners' inboxes. Phase B: owner sums its inbox slots in ascending order, updates
    // w and v, and stores the new w slice into every rank's replica; one flag barrier closes the step.
    const bool presum = c->fused_mode == 2;
    SS_TRY(ensure_fused(c, presum ? c->world : c->n));
    SS_TRY(ensure_dist_buffers(c));   // (sum_buf, rs_buf: NCCL mode only; allocated once)
    const uint32_t epA = ++c->epoch, epB = ++c->epoch;
    const int32_t me = c->rank;
    const int64_t lo = c->real_lo[me], cnt = c->real_hi[me] - lo;
    std::vector<std::pair<const float *, int32_t>> src;
    if (presum) {
      // one pass: pre-sum of the hosted gradients, each owner's slice stored into its inbox slot `me`
      ss::ScatterArgs sa;
      std::memset(&sa, 0, sizeof sa);
      sa.n_src = k;
      for (int32_t i = 0; i < k; ++i) {
        sa.src[i] = a.g[i];
        if (!aligned16(a.g[i])) return fail(c, SS_E_INVAL, "fused path needs 16-byte aligned gradients");
      }
      sa.slot[0] = me;
      for (int32_t q = 0; q < c->world; ++q) sa.inbox[q] = c->peer_inbox[q] + inbox_off(c);
      sa.reg_len = c->reg_len;
      sa.P = c->P;
      sa.sync = peer_sync(c, 0, epA, false, 1);
      Timed t;
      double remote = 0.0;
      for (int32_t q = 0; q < c->world; ++q)
        if (q != me) remote += (double)(c->real_hi[q] - c->real_lo[q]);
      timed_begin(c, &t, 3, 4.0 * ((double)c->P * k + (double)(c->real_hi[me] - lo)), 4.0 * remote);
      SS_CUDA(c, ss::launch_scatter_sum(sa, c->stream));
      timed_end(c, &t);
    } else {
      for (int32_t i = 0; i < k; ++i) src.push_back({a.g[i], ids[i]});
      SS_TRY(launch_scatter(c, src, epA));
    }
    const float *hosted_g[ss::kMaxWorkers];
    for (int32_t i = 0; i < k; ++i) hosted_g[i] = a.g[i];
    std::memset(a.g, 0, sizeof a.g);
    if (presum) {
      for (int32_t q = 0; q < c->world; ++q) a.g[q] = c->inbox + inbox_off(c) + (int64_t)q * c->reg_len;
      a.n_in = c->world;
    } else {
      int32_t ni = 0, h = 0;
      for (int32_t j = 0; j < c->n; ++j) {   // the members' slices, ascending worker order
        if (!c->member[j]) continue;
        a.g[ni++] = host_of(c, j) == me ? hosted_g[h++] + lo : c->inbox + inbox_off(c) + (int64_t)j * c->reg_len;
      }
      a.n_in = ni;
    }
    a.w = c->w + lo;
    a.v = c->v;
    a.count = cnt;
    a.n_bcast = 0;
    if (c->nvls.ready) {
      a.mc_w = (float *)c->nvls.mcv + lo;   // NVLS: one multicast store per element reaches every replica
    } else {
      for (int32_t step = 1; step < c->world; ++step)   // rotated: the ranks' stores go to distinct receivers
        a.bcast[a.n_bcast++] = c->peer_w[(me + step) % c->world] + lo;
    }
    a.sync = peer_sync(c, epA, epB, end_wait_needed(c, false), 2);
    Timed t;
    timed_begin(c, &t, 0, 4.0 * (double)cnt * (a.n_in + 4), 4.0 * (double)cnt * (c->nvls.ready ? 1 : a.n_bcast));
    SS_CUDA(c, ss::launch_bsp_update(a, vec, c->stream));
    timed_end(c, &t);
    c->xchg += 1;
  } else {
    SS_TRY(ensure_dist_buffers(c));
    if (k > 0) {
      ss::SumArgs s;
      std::memset(&s, 0, sizeof s);
      for (int32_t i = 0; i < k; ++i) s.g[i] = a.g[i];
      s.n_in = k;
      s.out = c->sum_buf;
      s.count = c->P;
      s.count_pad = c->P_pad;
      Timed t;
      timed_begin(c, &t, 2, 4.0 * ((double)c->P * k + (double)c->P_pad));
      SS_CUDA(c, ss::launch_local_sum(s, vec, c->stream));
      timed_end(c, &t);
    } else {
      SS_CUDA(c, cudaMemsetAsync(c->sum_buf, 0, (size_t)c->P_pad * sizeof(float), c->stream));
    }
    SS_NCCL(c, ncclReduceScatter(c->sum_buf, c->rs_buf, c->reg_len, ncclFloat, ncclSum, c->comm, c->stream));
    const int64_t lo = c->real_lo[c->rank], cnt = c->real_hi[c->rank] - lo;
    std::memset(a.g, 0, sizeof a.g);
    a.g[0] = c->rs_buf;
    a.n_in = 1;
    a.w = c->w + lo;
    a.v = c->v;
    a.count = cnt;
    Timed t;
    timed_begin(c, &t, 0, 4.0 * (double)cnt * 5);
    SS_CUDA(c, ss::launch_bsp_update(a, true, c->stream));
    timed_end(c, &t);
    SS_NCCL(c, ncclAllGather(c->w + (int64_t)c->rank * c->reg_len, c->w, c->reg_len, ncclFloat, c->comm,
                             c->stream));
  }
  SS_TRY(release_slots(c));
  for (int32_t j = 0; j < c->n; ++j)
    if (c->member[j]) record(c, j, c->version, 0);  // one staleness-0 record per BSP member
  c->version += 1;
  for (auto &b : c->base) b = c->version;
  return SS_OK;
}

ss_status ss_asp_push(ss_ctx *c, int32_t worker, const float *grad, int64_t version, int64_t *staleness_out) {
  SS_TRY(check_live(c));
  if (worker < 0 || worker >= c->n) return fail(c, SS_E_INVAL, "worker %d out of range", worker);
  const bool mine = host_of(c, worker) == c->rank;
  if (mine && !grad) return fail(c, SS_E_INVAL, "null gradient on the hosting rank");
  SS_TRY(maybe_switch(c));
  if (c->proto != SS_ASP) {
    c->dropped += 1;  // late in-flight push after ASP->BSP
    return fail(c, SS_E_STATE, "ss_asp_push under BSP (dropped)");
  }
  if (version > c->version || version < 0)
    return fail(c, SS_E_CAUSALITY, "base version %lld > current %lld", (long long)version, (long long)c->version);
  if (mine && c->world > 1 && c->fused_mode != 0 && !aligned16(grad) && !is_host_ptr(grad))
    return fail(c, SS_E_INVAL, "fused path needs 16-byte aligned gradients");
  Ev e{};
  e.kind = 0;
  e.worker = worker;
  e.lr = lr_at(c, c->version, SS_ASP);   // pre-increment version (reading C9)
  e.mu = asp_momentum(c, c->version);
  SS_TRY(enqueue_prepare(c, e, mine ? grad : nullptr, nullptr));   // may fail: nothing of this push applied yet
  enqueue_commit(c, e);
  const int64_t st = c->version - version;
  record(c, worker, version, st);
  c->version += 1;
  c->stepped = true;
  if (staleness_out) *staleness_out = st;
  return flush_if_full(c);
}

ss_status ss_pull(ss_ctx *c, int32_t worker, float *dst, int64_t *version_out) {
  SS_TRY(check_live(c));
  if (worker < 0 || worker >= c->n) return fail(c, SS_E_INVAL, "worker %d out of range", worker);
  const bool mine = host_of(c, worker) == c->rank;
  // SPMD rule: at G > 1 every pull moves data, so the hosting rank must name a destination (the others pass NULL
  // and send their owned slices).
  if (c->world > 1 && mine && !dst) return fail(c, SS_E_INVAL, "multi-GPU pull needs a destination");
  SS_TRY(maybe_switch(c));
  Ev e{};
  e.kind = 1;
  e.worker = worker;
  e.data = c->world > 1 || dst != nullptr;
  if (e.data) {
    SS_TRY(enqueue_prepare(c, e, nullptr, mine ? dst : nullptr));   // may fail: the base version is not moved yet
    enqueue_commit(c, e);
  }
  c->base[worker] = c->version;
  if (version_out) *version_out = c->version;
  return e.data ? flush_if_full(c) : SS_OK;
}

ss_status ss_switch(ss_ctx *c, int32_t proto, int64_t at_step) {
  SS_TRY(check_live(c));
  if (proto != SS_BSP && proto != SS_ASP) return fail(c, SS_E_INVAL, "bad protocol %d", proto);
  SS_TRY(maybe_switch(c));
  if (c->has_pending) return fail(c, SS_E_STATE, "a switch is already pending");
  c->has_pending = true;
  c->pending_proto = proto;
  c->pending_at = at_step;
  return maybe_switch(c);
}

ss_status ss_asp_replay(ss_ctx *c, const ss_event *ev, int64_t n_ev, int64_t *st_out) {
  if (!c || (!ev && n_ev > 0) || n_ev < 0) return SS_E_INVAL;
  for (int64_t i = 0; i < n_ev; ++i) {
    int64_t r = 0;
    ss_status s = ev[i].kind == 0 ? ss_asp_push(c, ev[i].worker, ev[i].grad, ev[i].version, &r)
                                  : ss_pull(c, ev[i].worker, ev[i].dst, &r);
    if (s != SS_OK) return s;
    if (st_out) st_out[i] = r;
  }
  return SS_OK;
}

ss_status ss_sync(ss_ctx *c) {
  SS_TRY(check_live(c));
  if (c->capturing) return fail(c, SS_E_STATE, "ss_sync inside a capture");
  return sync_impl(c);
}

ss_status ss_flush(ss_ctx *c) {
  SS_TRY(check_live(c));
  return flush(c);
}

// ---------------------------------------------------------------------------------------------------------------
// CUDA-graph capture of one step (latency-bound small models). The device work the calls
// between begin and end enqueue is recorded (not executed) into a graph; replay launches it K times and applies
// the host-state deltas the step produced (versions, base versions, staleness records, drops) K times.
ss_status ss_capture_begin(ss_ctx *c) {
  SS_TRY(check_live(c));
  if (c->capturing || c->prof) return fail(c, SS_E_STATE, "already capturing, or profiling is on");
  // G > 1: the exchange buffers, peer mappings and NVLS replica are set up by the first step (allocation and
  // synchronisation cannot be captured); the fused kernels take their flag epochs from a device counter, so the
  // graph replays with fresh epochs on every rank
  if (c->world > 1 && (c->fused_mode != 0 ? !c->ipc_ready : (c->sum_buf == nullptr ||
                                                              (int32_t)c->rslot.size() < c->max_win)))
    return fail(c, SS_E_STATE, "run one ordinary step before capturing (multi-GPU buffers are set up lazily)");
  SS_TRY(flush(c));
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  c->cap_v0 = c->version;
  c->cap_base0 = c->base;
  c->cap_log0 = (int64_t)c->log.size();
  c->cap_ddropped = c->dropped;
  c->cap_rel_since = c->version - c->asp_since;
  c->cap_epoch0 = c->epoch;
  c->cap_xchg0 = c->xchg;
  SS_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  c->capturing = true;
  return SS_OK;
}

ss_status ss_capture_end(ss_ctx *c, int64_t *version_delta) {
  if (!c || !c->capturing) return c ? fail(c, SS_E_STATE, "not capturing") : SS_E_INVAL;
  ss_status fl = flush(c);   // every queued window joins the graph
  if (fl == SS_OK && c->world > 1 && c->fused_mode != 0 && c->inbox_bufs == 2 && ((c->xchg - c->cap_xchg0) & 1)) {
    // an odd number of fused exchanges: consecutive replays would reuse one inbox buffer back to back, so the graph
    // closes with a cross-GPU barrier (an empty scatter launch that signals and waits for every rank)
    ss::ScatterArgs b;
    std::memset(&b, 0, sizeof b);
    for (int32_t q = 0; q < c->world; ++q) b.inbox[q] = c->peer_inbox[q];
    b.reg_len = c->reg_len;
    b.P = c->P;
    b.sync = peer_sync(c, 0, ++c->epoch, true, 0);
    cudaError_t le = ss::launch_scatter(b, c->stream);
    if (le != cudaSuccess) fl = fail(c, SS_E_CUDA, "capture barrier: %s", cudaGetErrorString(le));
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  c->capturing = false;
  if (fl != SS_OK) return fl;
  if (e != cudaSuccess) return fail(c, SS_E_CUDA, "capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&c->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(c, SS_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
  // the captured step already ran on the host side; its device work has not: run it once now
  SS_CUDA(c, cudaGraphLaunch(c->graph, c->stream));
  c->cap_dv = c->version - c->cap_v0;
  c->cap_depoch = c->epoch - c->cap_epoch0;
  c->cap_log.assign(c->log.begin() + c->cap_log0, c->log.end());
  c->cap_ddropped = c->dropped - c->cap_ddropped;
  if (version_delta) *version_delta = c->cap_dv;
  return SS_OK;
}

ss_status ss_capture_replay(ss_ctx *c, int64_t times) {
  SS_TRY(check_live(c));
  if (!c->graph || times < 0) return fail(c, SS_E_STATE, "no captured step");
  SS_TRY(maybe_switch(c));
  // validity: the step must leave the protocol where it found it (relative base versions, no pending switch), and
  // nothing the kernels baked in may change over the replayed versions (lr factor, momentum ramp)
  const int64_t dv = c->cap_dv;
  if (dv <= 0 || c->has_pending || c->win.size()) return fail(c, SS_E_STATE, "step not replayable");
  for (int32_t j = 0; j < c->n; ++j)
    if (c->base[j] - c->version != c->cap_base0[j] - c->cap_v0)
      return fail(c, SS_E_STATE, "base versions do not shift uniformly");
  const int64_t last = c->version + dv * times;
  for (int64_t b : c->bounds)
    if (b > c->cap_v0 && b < last) return fail(c, SS_E_STATE, "an lr boundary falls inside the replay");
  if (c->mom_rule != 0) return fail(c, SS_E_STATE, "a momentum ramp changes inside the replay");
  for (int64_t r = 0; r < times; ++r) {
    SS_CUDA(c, cudaGraphLaunch(c->graph, c->stream));
    const int64_t shift = c->version - c->cap_v0 - dv;   // version offset of this replay vs the captured step
    for (size_t i = 0; i + 3 < c->cap_log.size(); i += 4) {
      const int64_t st = c->cap_log[i + 2];
      if ((size_t)st >= c->hist.size()) c->hist.resize((size_t)st + 1, 0);
      c->hist[st] += 1;
      c->log.push_back(c->cap_log[i]);
      c->log.push_back(c->cap_log[i + 1] + shift + dv);
      c->log.push_back(st);
      c->log.push_back(c->cap_log[i + 3] + shift + dv);
    }
    c->version += dv;
    c->epoch += c->cap_depoch;         // the replayed kernels advanced the device epoch counter by as much
    c->dev_epoch += c->cap_depoch;
    for (auto &b : c->base) b += dv;
    c->dropped += c->cap_ddropped;
    if (c->asp_since >= c->cap_v0) c->asp_since += dv;   // the step switched to ASP: so does every replay
  }
  return SS_OK;
}

static ss_status gather_w(ss_ctx *c) {
  if (c->world == 1) return SS_OK;
  SS_NCCL(c, ncclAllGather(c->w + (int64_t)c->rank * c->reg_len, c->w, c->reg_len, ncclFloat, c->comm, c->stream));
  return SS_OK;
}

ss_status ss_read_params(ss_ctx *c, float *host_dst) {
  if (!c || !host_dst) return SS_E_INVAL;
  ss_status s = sync_impl(c);
  if (s != SS_OK && s != SS_E_DIVERGED) return s;
  SS_TRY(gather_w(c));
  SS_CUDA(c, cudaMemcpyAsync(host_dst, c->w, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  return s;
}

ss_status ss_read_velocity(ss_ctx *c, float *host_dst) {
  if (!c || !host_dst) return SS_E_INVAL;
  ss_status s = sync_impl(c);
  if (s != SS_OK && s != SS_E_DIVERGED) return s;
  if (c->world == 1) {
    SS_CUDA(c, cudaMemcpyAsync(host_dst, c->v, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
  } else {
    float *tmp = nullptr;
    SS_CUDA(c, cudaMallocAsync(&tmp, (size_t)c->P_pad * sizeof(float), c->stream));
    SS_NCCL(c, ncclAllGather(c->v, tmp, c->reg_len, ncclFloat, c->comm, c->stream));
    SS_CUDA(c, cudaMemcpyAsync(host_dst, tmp, (size_t)c->P * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    SS_CUDA(c, cudaFreeAsync(tmp, c->stream));
  }
  SS_CUDA(c, cudaStreamSynchronize(c->stream));
  return s;
}

ss_status ss_get_stats(ss_ctx *c, int64_t *version, int32_t *protocol, uint64_t *hist, int32_t hist_len,
                       uint64_t *dropped) {
  if (!c) return SS_E_INVAL;
  if (!c->diverged) SS_TRY(maybe_switch(c));
  if (version) *version = c->version;
  if (protocol) *protocol = c->proto;
  if (hist)
    for (int32_t i = 0; i < hist_len; ++i) hist[i] = (size_t)i < c->hist.size() ? c->hist[i] : 0;
  if (dropped) *dropped = c->dropped;
  return c->diverged ? SS_E_DIVERGED : SS_OK;
}

ss_status ss_get_log(ss_ctx *c, int64_t *rec4, int64_t cap, int64_t *total) {
  if (!c || cap < 0 || (cap > 0 && !rec4)) return SS_E_INVAL;
  const int64_t nrec = (int64_t)c->log.size() / 4;
  if (total) *total = nrec;
  const int64_t m = cap < nrec ? cap : nrec;
  if (m > 0) std::memcpy(rec4, c->log.data(), (size_t)m * 4 * sizeof(int64_t));
  return SS_OK;
}

ss_status ss_set_window(ss_ctx *c, int32_t max_events) {
  SS_TRY(check_live(c));
  if (max_events < 1 || max_events > ss::kMaxEvents) return fail(c, SS_E_INVAL, "window must be in [1, 64]");
  SS_TRY(flush(c));
  c->max_win = max_events;
  return SS_OK;
}

ss_status ss_set_fused(ss_ctx *c, int32_t mode) {
  SS_TRY(check_live(c));
  if (mode < 0 || mode > 3) return fail(c, SS_E_INVAL, "fused mode must be 0, 1, 2 or 3");
  SS_TRY(flush(c));
  c->fused_mode = mode;
  return SS_OK;
}

ss_status ss_get_exchange(ss_ctx *c, int32_t *mode, int32_t *nvls) {
  SS_TRY(check_live(c));
  if (mode) *mode = c->world > 1 ? c->fused_mode : 0;
  if (nvls) *nvls = c->nvls.ready ? 1 : 0;
  return SS_OK;
}

ss_status ss_pull_buffer(ss_ctx *c, int32_t worker, float **out) {
  SS_TRY(check_live(c));
  if (!out || worker < 0 || worker >= c->n) return fail(c, SS_E_INVAL, "bad worker or null output");
  if (c->world == 1 || c->fused_mode == 0) return fail(c, SS_E_STATE, "pull buffers exist in fused multi-GPU mode");
  if (host_of(c, worker) != c->rank) return fail(c, SS_E_INVAL, "worker %d is not hosted on this rank", worker);
  SS_TRY(ensure_fused(c, c->max_win));
  *out = c->pbuf + (int64_t)(worker - c->first_hosted) * c->P_pad;
  return SS_OK;
}

ss_status ss_grad_buffer(ss_ctx *c, int32_t worker, float **out) {
  SS_TRY(check_live(c));
  if (!out || worker < 0 || worker >= c->n) return fail(c, SS_E_INVAL, "bad worker or null output");
  if (c->world == 1 || c->fused_mode == 0) return fail(c, SS_E_STATE, "gradient buffers exist in fused multi-GPU mode");
  if (host_of(c, worker) != c->rank) return fail(c, SS_E_INVAL, "worker %d is not hosted on this rank", worker);
  SS_TRY(ensure_fused(c, c->max_win));
  *out = c->gbuf + (int64_t)(worker - c->first_hosted) * c->P_pad;
  return SS_OK;
}

ss_status ss_get_stream(ss_ctx *c, void **s) {
  if (!c || !s) return SS_E_INVAL;
  *s = c->stream;
  return SS_OK;
}

ss_status ss_wait_stream(ss_ctx *c, void *stream) {
  if (!c) return SS_E_INVAL;
  cudaEvent_t e;
  SS_CUDA(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  SS_CUDA(c, cudaEventRecord(e, (cudaStream_t)stream));
  SS_CUDA(c, cudaStreamWaitEvent(c->stream, e, 0));
  cudaEventDestroy(e);
  return SS_OK;
}

ss_status ss_profile(ss_ctx *c, int32_t on) {
  if (!c) return SS_E_INVAL;
  SS_TRY(drain_timed(c));
  c->prof = on != 0;
  if (on)
    for (auto &k : c->kstat) k = KStat{};
  return SS_OK;
}

ss_status ss_kernel_stats(ss_ctx *c, int32_t id, int64_t *launches, double *ms, double *bytes,
                          double *nvlink_bytes) {
  if (!c || id < 0 || id > 4) return SS_E_INVAL;
  SS_TRY(drain_timed(c));
  if (launches) *launches = c->kstat[id].launches;
  if (ms) *ms = c->kstat[id].ms;
  if (bytes) *bytes = c->kstat[id].bytes;
  if (nvlink_bytes) *nvlink_bytes = c->kstat[id].nvbytes;
  return SS_OK;
}

ss_status ss_synth_grad(uint64_t seed, int32_t j, int64_t k, int64_t i0, int64_t count, float *dst, void *stream) {
  if (!dst || j < 0 || j > 255 || k < 0 || k >= (int64_t(1) << 26) || i0 < 0 || count < 0 ||
      i0 + count > (int64_t(1) << 30))
    return SS_E_INVAL;
  return ss::launch_synth_grad(seed, j, k, i0, count, dst, (cudaStream_t)stream) == cudaSuccess ? SS_OK : SS_E_CUDA;
}

ss_status ss_dynamic_criterion(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const float *W,
                               const float *g_prev, float *g_out, float *stats, void *stream) {
  if (!X || !y || !W || !g_prev || !g_out || !stats || B < 2 || B > 1024 || d < 1 || C < 1 || C > 32)
    return SS_E_INVAL;
  cudaStream_t s = (cudaStream_t)stream;
  float *scratch = nullptr;
  double *part = nullptr;
  if (cudaMallocAsync(&scratch, ((size_t)B * (C + 1) + 1) * sizeof(float), s) != cudaSuccess) return SS_E_OOM;
  if (cudaMallocAsync(&part, (size_t)(B + 2) * sizeof(double), s) != cudaSuccess) return SS_E_OOM;
  cudaError_t e = ss::launch_dynamic_criterion(X, y, B, d, C, W, g_prev, g_out, stats, scratch, part, s);
  cudaFreeAsync(scratch, s);
  cudaFreeAsync(part, s);
  return e == cudaSuccess ? SS_OK : SS_E_CUDA;
}

ss_status ss_softmax_grad(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const float *W,
                          float *grad, float *loss, void *stream) {
  if (!X || !y || !W || !grad || !loss || B < 1 || B > 1024 || d < 1 || C < 1 || C > 32) return SS_E_INVAL;
  cudaStream_t s = (cudaStream_t)stream;
  float *scratch = nullptr;
  if (cudaMallocAsync(&scratch, (size_t)B * (C + 1) * sizeof(float), s) != cudaSuccess) return SS_E_OOM;
  cudaError_t e = ss::launch_softmax_grad(X, y, B, d, C, W, grad, loss, scratch, s);
  cudaFreeAsync(scratch, s);
  return e == cudaSuccess ? SS_OK : SS_E_CUDA;
}

}  // extern "C"

namespace ss {
CtxInfo ctx_info(const ss_ctx *c) {
  CtxInfo i;
  i.P = c->P;
  i.n = c->n;
  i.rank = c->rank;
  i.world = c->world;
  i.max_window = c->max_win;
  i.fused = c->fused_mode != 0;
  i.stream = c->stream;
  return i;
}

ss_status ctx_flush(ss_ctx *c) {
  SS_TRY(check_live(c));
  return flush(c);
}
}  // namespace ss
