// internal.h — launch interfaces shared by runtime.cu and kernels.cu (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "syncswitch.h"

namespace ss {

constexpr int kMaxWorkers = 256;  // SV §8b: workers in [1, 256]
constexpr int kMaxEvents = 64;    // events per ASP replay window
constexpr int kMaxPeers = 8;      // GPUs of one NVSwitch box

// Cross-GPU flag barrier over CUDA-IPC-mapped peer memory (fused path). Every rank owns
// sig_local[kMaxPeers] (written remotely by peers at index [their rank]) and a CTA completion counter. Epochs grow
// monotonically on every rank in the same SPMD order, so no flag is ever reset.
struct PeerSync {
  uint32_t *sig_local;              // this GPU's inbound flags
  uint32_t *sig_peer[kMaxPeers];    // rank q's sig_local (mapped; [rank] == sig_local)
  uint32_t *ctr;                    // CTA completion counter (local, returns to 0 after each use)
  int *err;                         // set when a wait times out (surfaced by ss_sync as SS_E_CUDA)
  int32_t rank, world;
  // Epochs are relative to this rank's device-resident counter *epoch_base (read at kernel entry, advanced by the last
  // CTA to the signalled epoch), so a captured CUDA graph replays with fresh epochs every time.
  uint32_t *epoch_base;
  int32_t has_wait;                 // every CTA waits for flag >= base + wait_off from all ranks before starting
  int32_t entry_signal;             // ... after signalling base + wait_off to every rank itself (the inputs this rank
                                    // contributes are ready at kernel entry: one-kernel pull exchange)
  uint32_t wait_off;
  uint32_t signal_off;              // !=0: the last CTA to finish signals every rank with base + signal_off
  int32_t end_wait;                 // and then waits until every rank has signalled it
  unsigned long long *trace;        // SS_TRACE: CTA 0 / the last CTA record globaltimer into trace[0..3] (or null)
};

// bsp_update (SV §2.5 K1): out-of-place aggregate of n_in inputs in ascending order, mean by `divisor`,
// momentum update of the owner slice. 1-GPU form: inputs = the n worker gradients, divisor = n. Post-reduce-scatter
// form: inputs = {reduce-scattered sum}, divisor = n. All pointers are pre-offset to the slice; `count` elements.
struct BspArgs {
  const float *g[kMaxWorkers];
  float *w;
  float *v;
  int *flag;          // set to 1 when a non-finite w or v is produced
  int64_t count;
  int32_t n_in;
  float divisor;
  float mu;
  float neg_eta;
  float lam;
  int32_t nesterov;         // 1: w -= eta * (g + mu * v_new) (ss_set_nesterov), else w -= eta * v_new
  float *bcast[kMaxPeers];  // fused path: remote replicas (at this slice's offset) that receive the updated w
  int32_t n_bcast;
  float *mc_w;              // NVLS: multicast view of this slice; one multimem.st updates every replica
  PeerSync sync;
};

// local_sum: out[i] = sum_{j ascending} g[j][i] for i < count, 0 for count <= i < count_pad (multi-GPU pre-sum
// of the workers hosted on one rank before the reduce-scatter).
struct SumArgs {
  const float *g[kMaxWorkers];
  float *out;
  int64_t count;
  int64_t count_pad;
  int32_t n_in;
};

// asp_replay (SV §2.5 K2): a window of events applied in order to one owner slice — ASP pushes and pulls
// and, on one GPU, BSP supersteps (the ascending sum of the barrier workers'
// gradients, the mean, the momentum update). Every event is elementwise, so one pass over the slice applies the whole
// window tile by tile with w and v held on chip: bit-identical to applying the events one after another.
constexpr int kMaxBspSrc = 128;                    // BSP gradients per window (all BSP events together)
constexpr int kMaxItems = kMaxEvents + kMaxBspSrc; // gradient tiles staged per tile of the slice
struct AspEvent {
  const float *src;   // push: gradient slice
  float *dst;         // pull: snapshot destination slice (nullptr: no data)
  float lr;           // push / BSP: eta at the event's (pre-increment) version
  float mu;           // push / BSP: momentum for this update (push: the post-switch momentum policy)
  float divisor;      // BSP: number of barrier workers (the mean is sum / divisor)
  int32_t kind;       // 0 push, 1 pull, 2 BSP superstep
  int32_t src0;       // BSP: its gradients are bsp_src[src0 .. src0 + n_src), ascending worker order
  int32_t n_src;
};
struct AspArgs {
  AspEvent ev[kMaxEvents];
  const float *bsp_src[kMaxBspSrc];
  float *w;
  float *v;
  int *flag;
  int64_t count;
  int32_t n_ev;
  int32_t tile;       // TMA form: floats per tile (multiple of 32, <= kTmaTile); set by launch_asp_replay
  int32_t n_item;     // TMA form: gradient sources per tile (pushes + BSP gradients; set by the launcher)
  int32_t stages;     // TMA form: ring depth in tiles (set by the launcher)
  float lam;
  int32_t nesterov;   // as BspArgs::nesterov
  PeerSync sync;
};

// scatter (fused path): copy every source's owner slices into the owners' inbox slots with posted NVLink stores:
// for each source k and each rank q != rank: src[k][real_lo[q] .. real_hi[q]) -> inbox[q] + slot[k]*reg_len.
struct ScatterArgs {
  const float *src[kMaxWorkers];
  int32_t slot[kMaxWorkers];
  float *inbox[kMaxPeers];
  int64_t reg_len;     // padded owner region (floats, multiple of 32): the slot stride and region size
  int64_t P;
  int32_t n_src;
  PeerSync sync;
};

constexpr int kSigWords = 256;   // flag block (uint32): [0..7] inbound epoch flags, [32] CTA counter, [64] timeout
                                 // flag, [160] device epoch counter

// What the in-library drivers (scenario.cpp) need to know about a context.
struct CtxInfo {
  int64_t P;
  int32_t n, rank, world, max_window;
  bool fused;
  cudaStream_t stream;
};

cudaError_t launch_bsp_update(const BspArgs &a, bool vec, cudaStream_t s);
cudaError_t launch_local_sum(const SumArgs &a, bool vec, cudaStream_t s);
cudaError_t launch_asp_replay(const AspArgs &a, bool vec, cudaStream_t s);
cudaError_t launch_scatter(const ScatterArgs &a, cudaStream_t s);
cudaError_t launch_scatter_sum(const ScatterArgs &a, cudaStream_t s);
cudaError_t launch_synth_grad(uint64_t seed, int32_t j, int64_t k, int64_t i0, int64_t count, float *dst,
                              cudaStream_t s);
cudaError_t launch_dynamic_criterion(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C,
                                     const float *W, const float *g_prev, float *g_out, float *stats, float *scratch,
                                     double *part, cudaStream_t s);
cudaError_t launch_softmax_grad(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const float *W,
                                float *grad, float *loss, float *scratch, cudaStream_t s);

}  // namespace ss

struct ss_ctx;
namespace ss {
CtxInfo ctx_info(const ss_ctx *c);
// Launches the pending window (the device work of already accepted calls); no-op when nothing is pending.
ss_status ctx_flush(ss_ctx *c);
}  // namespace ss
