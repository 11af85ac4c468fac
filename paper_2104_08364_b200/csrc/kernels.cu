// kernels.cu — sm_100a kernels of the Sync-Switch synchronization path.
//
//   bsp_update   (K1) fused aggregate + mean + momentum update of an owner slice
//   local_sum    (K1a) ascending pre-sum of the workers hosted on one rank (G > 1)
//   asp_replay   (K2) a window of ASP pushes/pulls applied in arrival order
//   synth_grad   (K3) seeded counter-hash gradients                      —
//   softmax_grad (K4) toy softmax-regression loss and gradient (SURVEY config 1)     P:1072 (worker fwd/bwd)
//
// The path is HBM-bound streaming (arithmetic intensity ~0.25 flop/B, no contraction): no tensor cores. Every
// kernel moves 128-bit vectors with streaming cache hints, keeps many independent loads in flight per thread
// (all inputs of a chunk are issued before the dependent arithmetic), and runs a grid sized to the SM count.
// Floating-point order is fixed and explicit (__fadd_rn / __fmaf_rn / __fdiv_rn) so that results are bit-identical
// to the CPU oracle's written order (reading C12): sum in ascending worker order, then the mean, then
// v = fma(mu, v, g), w = fma(-eta, v, w).
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "internal.h"

namespace ss {
namespace {

constexpr int kThreads = 256;

// Streaming 128-bit accesses: loads cached in L2 only (.cg — never a stale L1 line for data written by peers),
// stores marked evict-first (.cs).
__device__ __forceinline__ float4 ld4(const float *p) { return __ldcg(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ void st4(float *p, float4 x) { __stcs(reinterpret_cast<float4 *>(p), x); }

// Programmatic dependent launch (the streaming kernels are launched with programmatic stream serialization): a
// kernel lets the next one on the stream be scheduled as soon as all of its CTAs are resident (trigger), and reads
// nothing another kernel wrote before griddepcontrol.wait returns — which is when the previous grid has completed and
// its memory operations are visible. The next launch's scheduling and prologue then overlap this kernel's tail.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------------------------------------------------------
// Cross-GPU flag barrier (fused path). Release/acquire at system scope over NVLink-mapped peer memory; every wait
// is bounded (kTimeoutNs) so a missing peer can never hang the GPU: the wait gives up and raises *err.
constexpr unsigned long long kTimeoutNs = 10ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block-wide: returns when every rank has signalled >= epoch (or on timeout).
// SS_TRACE timestamps (globaltimer ns) of one fused launch: [0] CTA 0 entered, [1] CTA 0's start wait satisfied,
// [2] the last CTA about to signal, [3] the last CTA's end wait satisfied.
__device__ __forceinline__ void trace_mark(const PeerSync &s, int k) {
  if (s.trace != nullptr && threadIdx.x == 0) s.trace[k] = globaltimer();
}

__device__ void peer_wait(const PeerSync &s, uint32_t epoch) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = globaltimer();
    bool timed_out = false;
    for (int q = 0; q < s.world && !timed_out; ++q) {
      while ((int32_t)(ld_acquire_sys(s.sig_local + q) - epoch) < 0) {
        if (globaltimer() - t0 > kTimeoutNs) {
          atomicExch(s.err, 1);
          timed_out = true;
          break;
        }
        __nanosleep(100);
      }
    }
  }
  __syncthreads();
}

// Absolute epochs of this launch: the rank's device counter (advanced by the previous fused kernel) + the offsets.
struct Ep {
  uint32_t wait, signal;
};
__device__ __forceinline__ Ep peer_epochs(const PeerSync &s) {
  const uint32_t b = s.epoch_base ? *reinterpret_cast<const volatile uint32_t *>(s.epoch_base) : 0u;
  return Ep{b + s.wait_off, s.signal_off ? b + s.signal_off : 0u};
}

// Block-wide, at kernel entry: CTA 0 stamps trace[0]; every CTA waits for the wait epoch when set (CTA 0 stamps
// trace[1]). Returns the launch's epochs.
__device__ __forceinline__ Ep peer_enter(const PeerSync &s) {
  const Ep ep = peer_epochs(s);
  if (blockIdx.x == 0) trace_mark(s, 0);
  if (s.has_wait) {
    if (s.entry_signal && threadIdx.x == 0) {   // every CTA (idempotent): no CTA waits on one not yet resident
      __threadfence_system();
      for (int q = 0; q < s.world; ++q) st_release_sys(s.sig_peer[q] + s.rank, ep.wait);
    }
    peer_wait(s, ep.wait);
    if (blockIdx.x == 0) trace_mark(s, 1);
  }
  return ep;
}

// Block-wide, at kernel end: the last CTA of the grid publishes the signal epoch to every rank (after a system-scope
// fence that orders all of this grid's stores, local and remote, before the flag), advances the rank's epoch counter
// to it, and optionally waits for all ranks.
__device__ void peer_done(const PeerSync &s, const Ep &ep) {
  if (ep.signal == 0) return;
  __threadfence_system();
  __syncthreads();
  __shared__ uint32_t last;
  if (threadIdx.x == 0) last = atomicAdd(s.ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) {
    *s.ctr = 0;
    __threadfence_system();
    trace_mark(s, 2);
    for (int q = 0; q < s.world; ++q) st_release_sys(s.sig_peer[q] + s.rank, ep.signal);
    *s.epoch_base = ep.signal;   // every CTA of this grid read the base at entry; the next kernel sees the new one
  }
  if (s.end_wait) {
    peer_wait(s, ep.signal);
    trace_mark(s, 3);
  }
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ bool nonfinite(float x) { return !isfinite(x); }

// NVLS: one store through the multicast view writes the value into every GPU's copy (switch replication).
__device__ __forceinline__ void mc_st4(float *p, float4 x) {
  asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(x.x), "f"(x.y), "f"(x.z),
               "f"(x.w)
               : "memory");
}
__device__ __forceinline__ void mc_st1(float *p, float x) {
  asm volatile("multimem.st.weak.global.f32 [%0], %1;" ::"l"(p), "f"(x) : "memory");
}

// g = a / divisor (+ lam*w); v = mu*v + g; w = w - eta*v.  When the divisor is a power of two, a*recip is the same
// correctly rounded quotient, so `use_recip` changes no bit.
struct Upd {
  float divisor, recip, mu, neg_eta, lam;
  bool use_recip;
  bool nesterov;
  __device__ __forceinline__ void operator()(float a, float &w, float &v) const {
    float g = use_recip ? __fmul_rn(a, recip) : __fdiv_rn(a, divisor);
    if (lam != 0.0f) g = __fmaf_rn(lam, w, g);
    v = __fmaf_rn(mu, v, g);
    w = __fmaf_rn(neg_eta, nesterov ? __fmaf_rn(mu, v, g) : v, w);   // Nesterov: step along g + mu*v_new
  }
};

__device__ __forceinline__ bool is_pow2(float d) {
  int e;
  return frexpf(d, &e) == 0.5f;
}

// ---------------------------------------------------------------------------------------------------------------
// K1 bsp_update
#ifndef SS_BSP_U
#define SS_BSP_U 2          // tuning knobs (tools/kernel_sweep.py builds variants)
#endif
#ifndef SS_BSP_G
#define SS_BSP_G 8
#endif
constexpr int kU1 = SS_BSP_U;  // float4 chunks per thread per iteration
constexpr int kG1 = SS_BSP_G;  // gradients loaded together

// U float4 per thread per iteration, GL gradients loaded together (the streaming form uses the sweep's kU1/kG1; a
// launch smaller than one wave of it uses <1, 4>: profiles/r01_bsp_sweep.txt, config 2)
template <bool VEC, int U = kU1, int GL = kG1>
__global__ void __launch_bounds__(kThreads) bsp_update_kernel(const __grid_constant__ BspArgs a) {
  pdl_trigger();
  pdl_wait();
  const Ep ep = peer_enter(a.sync);
  const Upd up{a.divisor, 1.0f / a.divisor, a.mu, a.neg_eta, a.lam, is_pow2(a.divisor), a.nesterov != 0};
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  if (VEC) {
    const int64_t n4 = a.count >> 2;
    for (int64_t q0 = tid; q0 < n4; q0 += stride * U) {
      float4 acc[U], wv[U], vv[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = q0 + u * stride;
        ok[u] = q < n4;
        if (ok[u]) {
          acc[u] = ld4(a.g[0] + 4 * q);
          wv[u] = ld4(a.w + 4 * q);
          vv[u] = ld4(a.v + 4 * q);
        }
      }
      for (int j0 = 1; j0 < a.n_in; j0 += GL) {
        float4 t[GL][U];
#pragma unroll
        for (int jj = 0; jj < GL; ++jj)
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j0 + jj < a.n_in && ok[u]) t[jj][u] = ld4(a.g[j0 + jj] + 4 * (q0 + u * stride));
#pragma unroll
        for (int jj = 0; jj < GL; ++jj)
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (j0 + jj < a.n_in && ok[u]) acc[u] = add4(acc[u], t[jj][u]);  // ascending worker order
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!ok[u]) continue;
        up(acc[u].x, wv[u].x, vv[u].x);
        up(acc[u].y, wv[u].y, vv[u].y);
        up(acc[u].z, wv[u].z, vv[u].z);
        up(acc[u].w, wv[u].w, vv[u].w);
        bad |= nonfinite(wv[u].x) | nonfinite(wv[u].y) | nonfinite(wv[u].z) | nonfinite(wv[u].w) |
               nonfinite(vv[u].x) | nonfinite(vv[u].y) | nonfinite(vv[u].z) | nonfinite(vv[u].w);
        const int64_t q = q0 + u * stride;
        if (a.mc_w) {
          mc_st4(a.mc_w + 4 * q, wv[u]);        // NVLS: every replica, this GPU's included ...
          st4(a.w + 4 * q, wv[u]);              // ... and the authoritative copy directly (later local reads)
        } else {
          st4(a.w + 4 * q, wv[u]);
          for (int b = 0; b < a.n_bcast; ++b)   // fused path: the updated slice goes straight to every replica
            *reinterpret_cast<float4 *>(a.bcast[b] + 4 * q) = wv[u];
        }
        st4(a.v + 4 * q, vv[u]);
      }
    }
    // scalar tail (count % 4 elements)
    const int64_t i = 4 * n4 + tid;
    if (i < a.count) {
      float acc = a.g[0][i];
      for (int j = 1; j < a.n_in; ++j) acc = __fadd_rn(acc, a.g[j][i]);
      float w = a.w[i], v = a.v[i];
      up(acc, w, v);
      bad |= nonfinite(w) | nonfinite(v);
      if (a.mc_w) mc_st1(a.mc_w + i, w);
      a.w[i] = w;
      if (!a.mc_w)
        for (int b = 0; b < a.n_bcast; ++b) a.bcast[b][i] = w;
      a.v[i] = v;
    }
  } else {
    for (int64_t i = tid; i < a.count; i += stride) {
      float acc = a.g[0][i];
      for (int j = 1; j < a.n_in; ++j) acc = __fadd_rn(acc, a.g[j][i]);
      float w = a.w[i], v = a.v[i];
      up(acc, w, v);
      bad |= nonfinite(w) | nonfinite(v);
      if (a.mc_w) mc_st1(a.mc_w + i, w);
      a.w[i] = w;
      if (!a.mc_w)
        for (int b = 0; b < a.n_bcast; ++b) a.bcast[b][i] = w;
      a.v[i] = v;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *a.flag = 1;
  if (a.mc_w) asm volatile("fence.proxy.alias;" ::: "memory");  // multicast stores before unicast accesses
  peer_done(a.sync, ep);
}

// ---------------------------------------------------------------------------------------------------------------
// K1a local_sum
template <bool VEC>
__global__ void __launch_bounds__(kThreads) local_sum_kernel(const __grid_constant__ SumArgs a) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (VEC) {
    const int64_t n4 = a.count >> 2;
    for (int64_t q0 = tid; q0 < n4; q0 += stride * kU1) {
      float4 acc[kU1];
      bool ok[kU1];
#pragma unroll
      for (int u = 0; u < kU1; ++u) {
        const int64_t q = q0 + u * stride;
        ok[u] = q < n4;
        if (ok[u]) acc[u] = ld4(a.g[0] + 4 * q);
      }
      for (int j0 = 1; j0 < a.n_in; j0 += kG1) {
        float4 t[kG1][kU1];
#pragma unroll
        for (int jj = 0; jj < kG1; ++jj)
#pragma unroll
          for (int u = 0; u < kU1; ++u)
            if (j0 + jj < a.n_in && ok[u]) t[jj][u] = ld4(a.g[j0 + jj] + 4 * (q0 + u * stride));
#pragma unroll
        for (int jj = 0; jj < kG1; ++jj)
#pragma unroll
          for (int u = 0; u < kU1; ++u)
            if (j0 + jj < a.n_in && ok[u]) acc[u] = add4(acc[u], t[jj][u]);
      }
#pragma unroll
      for (int u = 0; u < kU1; ++u)
        if (ok[u]) st4(a.out + 4 * (q0 + u * stride), acc[u]);
    }
    done = 4 * n4;
  }
  for (int64_t i = done + tid; i < a.count_pad; i += stride) {
    float acc = 0.0f;
    if (i < a.count) {
      acc = a.g[0][i];
      for (int j = 1; j < a.n_in; ++j) acc = __fadd_rn(acc, a.g[j][i]);
    }
    a.out[i] = acc;
  }
}

// ---------------------------------------------------------------------------------------------------------------
// K2 asp_replay, scalar form: used only when a gradient or snapshot pointer is not 16-byte aligned (the TMA form
// below needs 16-byte aligned sources). Same arithmetic, element by element: every event updates w, v in window order
// and every pull stores the current w — so a pull observes exactly the updates before it, on every shard (C6).
__global__ void __launch_bounds__(kThreads) asp_replay_scalar_kernel(const __grid_constant__ AspArgs a) {
  const Ep ep = peer_enter(a.sync);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const float lam = a.lam;
  const bool nest = a.nesterov != 0;
  bool bad = false;
  for (int64_t i = tid; i < a.count; i += stride) {
    float w = a.w[i], v = a.v[i];
    for (int e = 0; e < a.n_ev; ++e) {
      const AspEvent &x = a.ev[e];
      if (x.kind == 0) {
        float g = x.src[i];
        if (lam != 0.0f) g = __fmaf_rn(lam, w, g);   // g + f(w) at the PS's current w
        v = __fmaf_rn(x.mu, v, g);                    // per-push momentum (post-switch policy)
        w = __fmaf_rn(-x.lr, nest ? __fmaf_rn(x.mu, v, g) : v, w);
      } else if (x.kind == 2) {
        float acc = a.bsp_src[x.src0][i];
        for (int k = 1; k < x.n_src; ++k) acc = __fadd_rn(acc, a.bsp_src[x.src0 + k][i]);   // ascending workers
        const Upd up{x.divisor, 1.0f / x.divisor, x.mu, -x.lr, lam, is_pow2(x.divisor), nest};
        up(acc, w, v);
      } else if (x.dst) {
        x.dst[i] = w;
      }
    }
    bad |= nonfinite(w) | nonfinite(v);
    a.w[i] = w;
    a.v[i] = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *a.flag = 1;
  peer_done(a.sync, ep);
}

// ---------------------------------------------------------------------------------------------------------------
// K2, TMA form: the same replay, with every push's gradient tile staged through a shared-memory ring filled by 1-D
// bulk copies (cp.async.bulk, completion on an mbarrier). One CTA walks its tiles (kTmaTile floats = 8 KB); the w and
// v of a tile live in registers for the whole window; thread 0 keeps kTmaStages tile loads in flight ahead of the
// consumers, across push and tile boundaries, so the bytes in flight no longer depend on registers per thread.
#ifndef SS_TMA_TILE
#define SS_TMA_TILE 2048   // tuning knobs (tools/kernel_sweep.py builds variants)
#endif
#ifndef SS_TMA_STAGES
#define SS_TMA_STAGES 10   // 80 KB rings -> 2 CTAs per SM: 96.5-98% of the HBM copy vs 93% at 6 stages / 4 CTAs
#endif                     // (profiles/r01_replay_sweep.txt)
constexpr int kTmaTile = SS_TMA_TILE;                // floats per tile (max): 256 threads x 2 float4
constexpr int kTmaStages = SS_TMA_STAGES;
constexpr int kTmaSmem = kTmaStages * kTmaTile * 4;  // 80 KB of dynamic shared memory
constexpr int kTU = kTmaTile / (4 * kThreads);       // float4 per thread per tile
constexpr int kMaxStages = kMaxItems;                // ring stages (runtime; the small-launch form holds every item)
constexpr int kTmaSmemMax = 200 * 1024;              // dynamic shared memory the launcher may ask for
static_assert(kTU >= 1 && kTmaTile % (4 * kThreads) == 0, "tile must be a multiple of 4 x kThreads floats");

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// kRefill = false: every CTA's items (tiles x gradient sources) fit the ring, so no stage is ever reused and the
// per-item CTA barrier is dropped (small P; a separate instantiation because a runtime-conditional barrier costs the
// large-P loop 2.5%: profiles/r01_replay_condsync.txt). Tile length (a.tile floats) and ring depth (a.stages) are
// chosen per launch: the streaming form uses kTmaTile-float tiles and a kTmaStages ring; a launch smaller than a few
// waves of it (config 2) uses one shorter tile per CTA and a ring deep enough for all of that tile's gradient sources,
// so every CTA issues all its bulk copies at once and never waits on a CTA barrier.
// Window events: push (one staged gradient tile), BSP superstep (n_src staged tiles summed in ascending worker order
// into a register accumulator, then the mean and the momentum update), pull (store of the current w).
template <bool kRefill>
__global__ void __launch_bounds__(kThreads) asp_replay_tma_kernel(const __grid_constant__ AspArgs a) {
  pdl_trigger();
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ const float *item_src[kMaxItems];
  struct SEv {                                               // the window's events, copied once per CTA: the event
    float *dst;                                              // loop reads shared memory instead of indexing the
    float lr, mu, divisor;                                   // kernel parameters at a run-time index
    int32_t kind, n_src;
  };
  __shared__ SEv sev[kMaxEvents];
  // ring depth and tile length: compile-time in the streaming (refill) form, per launch in the small-launch form
  const int n_stage = kRefill ? kTmaStages : a.stages;      // (<= kMaxStages)
  const float lam = a.lam;
  const bool nest = a.nesterov != 0;
  const int n_item = a.n_item;                               // gradient sources per tile, in event order
  const int64_t nvec = (a.count >> 2) << 2;                  // elements covered by 16-byte tiles
  const int64_t tsz = kRefill ? (int64_t)kTmaTile : (int64_t)a.tile;   // floats per tile (<= kTmaTile)
  const int64_t n_tiles = (nvec + tsz - 1) / tsz;
  const int64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t items = my_tiles * n_item;                   // one gradient tile per (tile, source)

  // w and v of the CTA's current tile live in registers; the first tile's loads are issued before the prologue so
  // their latency overlaps it, each later tile's right after the previous one is stored
  float4 wv[kTU], vv[kTU];
  bool ok[kTU];
  auto load_wv = [&](int64_t tl) {
    const int64_t off = (blockIdx.x + tl * gridDim.x) * tsz;
    const int64_t len = min(tsz, nvec - off);
#pragma unroll
    for (int u = 0; u < kTU; ++u) {
      const int64_t i = 4 * (threadIdx.x + u * kThreads);    // element within the tile
      ok[u] = i < len;
      if (ok[u]) {
        wv[u] = ld4(a.w + off + i);
        vv[u] = ld4(a.v + off + i);
      }
    }
  };
  // Prologue, warp 0 (kernel parameters and shared memory only, so it overlaps the previous kernel's tail): list the gradient sources of a tile in event order (lane l takes events l and l + 32; their
  // item offsets are a warp prefix sum of the per-event source counts) and initialise the ring's barriers.
  static_assert(kMaxEvents <= 64, "two events per lane");
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    auto count_of = [&](int e) {
      return e < a.n_ev ? (a.ev[e].kind == 0 ? 1 : a.ev[e].kind == 2 ? a.ev[e].n_src : 0) : 0;
    };
    const int c0 = count_of(lane), c1 = count_of(lane + 32);
    int s0 = c0, s1 = c1;                                    // inclusive scans over the lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t0 = __shfl_up_sync(0xffffffffu, s0, d), t1 = __shfl_up_sync(0xffffffffu, s1, d);
      if (lane >= d) {
        s0 += t0;
        s1 += t1;
      }
    }
    const int tot0 = __shfl_sync(0xffffffffu, s0, 31);
    auto list = [&](int e, int pos, int cnt) {
      for (int k = 0; k < cnt; ++k)
        item_src[pos + k] = a.ev[e].kind == 0 ? a.ev[e].src : a.bsp_src[a.ev[e].src0 + k];
    };
    list(lane, s0 - c0, c0);
    list(lane + 32, tot0 + s1 - c1, c1);
    if (kRefill)   // (streaming form: config 3 asp_replay 333 -> 327 us; the short small-launch form loses more in the copy)
      for (int e = lane; e < a.n_ev; e += 32)
        sev[e] = SEv{a.ev[e].dst, a.ev[e].lr, a.ev[e].mu, a.ev[e].divisor, a.ev[e].kind, a.ev[e].n_src};
    for (int st = lane; st < n_stage; st += 32) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();                                                // from here on: data of earlier kernels
  const Ep ep = peer_enter(a.sync);
  // the bulk copies below (async proxy) may read slices peers wrote before the flag this CTA acquired (generic
  // proxy): order them after the acquire
  if (a.sync.has_wait && threadIdx.x < 32) asm volatile("fence.proxy.async.global;" ::: "memory");
  if (my_tiles > 0) load_wv(0);
  __syncthreads();

  // Items are staged and consumed in order, so both sides walk cursors instead of dividing by the runtime ring depth
  // and source count: the producer (thread 0) keeps (tile, source, stage) of the next item to issue; every thread
  // keeps (stage, parity) of the next item to consume.
  int64_t p_next = 0, p_tile = blockIdx.x;                   // producer cursor (thread 0 only)
  int p_src = 0, p_stage = 0;
  auto issue_next = [&]() {                                  // thread 0: stage the gradient tile of item p_next
    const int64_t off = p_tile * tsz;
    const int64_t len = min(tsz, nvec - off);
    mbar_expect_tx(&full[p_stage], (uint32_t)(len * 4));
    bulk_g2s(ring + p_stage * tsz, item_src[p_src] + off, (uint32_t)(len * 4), &full[p_stage]);
    ++p_next;
    if (++p_src == n_item) {
      p_src = 0;
      p_tile += gridDim.x;
    }
    if (++p_stage == n_stage) p_stage = 0;
  };
  if (kRefill) {
    if (threadIdx.x == 0)
      while (p_next < items && p_next < n_stage) issue_next();
  } else if (threadIdx.x < 32) {                             // the ring holds every item: warp 0 issues them all
    for (int64_t it = threadIdx.x; it < items; it += 32) {
      const int64_t off = (blockIdx.x + (it / n_item) * gridDim.x) * tsz;
      const int64_t len = min(tsz, nvec - off);
      mbar_expect_tx(&full[it], (uint32_t)(len * 4));
      bulk_g2s(ring + it * tsz, item_src[it % n_item] + off, (uint32_t)(len * 4), &full[it]);
    }
  }
  int c_stage = 0;                                           // consumer cursor: stage and parity of item `it`
  uint32_t c_phase = 0;
  auto wait_item = [&]() { mbar_wait(&full[c_stage], c_phase); };
  // the thread's float4 u of the staged tile of the item being consumed
  auto staged = [&](int u) -> float4 {
    return *reinterpret_cast<const float4 *>(ring + c_stage * tsz + 4 * (threadIdx.x + u * kThreads));
  };
  auto release = [&]() {                                     // done with the item being consumed; advance
    if (kRefill) {                                           // (a window that fits the ring never reuses a stage)
      __syncthreads();                                       // every thread is done with this stage
      if (threadIdx.x == 0 && p_next < items) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_next();                                        // refills exactly this stage (p_next = it + n_stage)
      }
    }
    if (++c_stage == n_stage) {
      c_stage = 0;
      c_phase ^= 1u;
    }
  };

  bool bad = false;
  for (int64_t tl = 0; tl < my_tiles; ++tl) {
    const int64_t off = (blockIdx.x + tl * gridDim.x) * tsz;
    for (int e = 0; e < a.n_ev; ++e) {
      // event fields: the shared copy in the streaming form, the kernel parameters (read only where used) otherwise
#define EVF(f) (kRefill ? sev[e].f : a.ev[e].f)
      const int kind = EVF(kind);
      if (kind == 0) {
        wait_item();
        const float neg_eta = -EVF(lr), mu = EVF(mu);
#pragma unroll
        for (int u = 0; u < kTU; ++u) {
          if (!ok[u]) continue;
          float4 g = staged(u);
          float *gp = &g.x, *wp = &wv[u].x, *vp = &vv[u].x;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float gg = gp[c];
            if (lam != 0.0f) gg = __fmaf_rn(lam, wp[c], gg);   // g + f(w) at the PS's current w
            vp[c] = __fmaf_rn(mu, vp[c], gg);
            wp[c] = __fmaf_rn(neg_eta, nest ? __fmaf_rn(mu, vp[c], gg) : vp[c], wp[c]);
          }
        }
        release();
      } else if (kind == 2) {
        float4 acc[kTU];
        const int ns = EVF(n_src);
        for (int k = 0; k < ns; ++k) {
          wait_item();
#pragma unroll
          for (int u = 0; u < kTU; ++u) {
            if (!ok[u]) continue;
            const float4 g = staged(u);
            acc[u] = k == 0 ? g : add4(acc[u], g);            // ascending worker order (reading C12)
          }
          release();
        }
        const float dv = EVF(divisor);
        const Upd up{dv, 1.0f / dv, EVF(mu), -EVF(lr), lam, is_pow2(dv), nest};
#pragma unroll
        for (int u = 0; u < kTU; ++u) {
          if (!ok[u]) continue;
          up(acc[u].x, wv[u].x, vv[u].x);
          up(acc[u].y, wv[u].y, vv[u].y);
          up(acc[u].z, wv[u].z, vv[u].z);
          up(acc[u].w, wv[u].w, vv[u].w);
        }
      } else if (EVF(dst) != nullptr) {
        float *const dst = EVF(dst);
#pragma unroll
        for (int u = 0; u < kTU; ++u)
          if (ok[u]) st4(dst + off + 4 * (threadIdx.x + u * kThreads), wv[u]);
      }
    }
#undef EVF
#pragma unroll
    for (int u = 0; u < kTU; ++u) {
      if (!ok[u]) continue;
      bad |= nonfinite(wv[u].x) | nonfinite(wv[u].y) | nonfinite(wv[u].z) | nonfinite(wv[u].w) |
             nonfinite(vv[u].x) | nonfinite(vv[u].y) | nonfinite(vv[u].z) | nonfinite(vv[u].w);
      const int64_t i = off + 4 * (threadIdx.x + u * kThreads);
      st4(a.w + i, wv[u]);
      st4(a.v + i, vv[u]);
    }
    if (tl + 1 < my_tiles) load_wv(tl + 1);
  }
  // scalar tail (count % 4 elements), first CTA
  if (blockIdx.x == 0) {
    const int64_t i = nvec + threadIdx.x;
    if (i < a.count) {
      float w = a.w[i], v = a.v[i];
      for (int e = 0; e < a.n_ev; ++e) {
        const AspEvent &x = a.ev[e];
        if (x.kind == 0) {
          float gg = x.src[i];
          if (lam != 0.0f) gg = __fmaf_rn(lam, w, gg);
          v = __fmaf_rn(x.mu, v, gg);
          w = __fmaf_rn(-x.lr, nest ? __fmaf_rn(x.mu, v, gg) : v, w);
        } else if (x.kind == 2) {
          float acc = a.bsp_src[x.src0][i];
          for (int k = 1; k < x.n_src; ++k) acc = __fadd_rn(acc, a.bsp_src[x.src0 + k][i]);
          const Upd up{x.divisor, 1.0f / x.divisor, x.mu, -x.lr, lam, is_pow2(x.divisor), nest};
          up(acc, w, v);
        } else if (x.dst) {
          x.dst[i] = w;
        }
      }
      bad |= nonfinite(w) | nonfinite(v);
      a.w[i] = w;
      a.v[i] = v;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *a.flag = 1;
  peer_done(a.sync, ep);
}

// ---------------------------------------------------------------------------------------------------------------
// scatter (fused path): every hosted gradient's owner slices go to the owners' inboxes with
// posted 128-bit NVLink stores (the local slice is read in place by the owner update, never copied).
__global__ void __launch_bounds__(kThreads) scatter_kernel(const __grid_constant__ ScatterArgs a) {
  pdl_trigger();
  pdl_wait();
  const Ep ep = peer_enter(a.sync);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int me = a.sync.rank, G = a.sync.world;
  constexpr int U = 8;  // stores in flight per thread (posted NVLink writes; the loads come from local HBM)
  for (int k = 0; k < a.n_src; ++k) {
    // one contiguous segment per (source, destination rank), no per-element division; destinations in rotated order
    // (me+1, me+2, ...) so that at any moment the ranks write to distinct receivers instead of all hitting one ingress
    for (int step = 1; step < G; ++step) {
      const int r = (me + step) % G;
      const int64_t lo = min((int64_t)r * a.reg_len, a.P), cnt = min((int64_t)(r + 1) * a.reg_len, a.P) - lo;
      const float *src = a.src[k] + lo;
      float *dst = a.inbox[r] + (int64_t)a.slot[k] * a.reg_len;
      const int64_t n4 = cnt >> 2;
      for (int64_t q0 = tid; q0 < n4; q0 += stride * U) {
        float4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q0 + u * stride < n4) x[u] = ld4(src + 4 * (q0 + u * stride));
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (q0 + u * stride < n4) *reinterpret_cast<float4 *>(dst + 4 * (q0 + u * stride)) = x[u];
      }
      const int64_t i = 4 * n4 + tid;  // scalar tail
      if (i < cnt) dst[i] = src[i];
    }
  }
  peer_done(a.sync, ep);
}

// scatter_sum (fused mode 2): one pass over the hosted gradients — sum them in ascending order and store each owner's
// slice of the pre-sum straight into that owner's inbox slot a.slot[0] (this rank's id); the own slice stays local.
// The grid is split into G interleaved CTA subsets, subset k serving destination region (me + 1 + k) % G: the NVLink
// stores to every peer and the local-only pass over the own region run at the same time (processing the regions one
// after another left the own region's HBM pass on the critical path after the NVLink-bound ones).
constexpr int kScsU = 2;   // float4 chunks per thread per iteration
__global__ void __launch_bounds__(kThreads) scatter_sum_kernel(const __grid_constant__ ScatterArgs a) {
  pdl_trigger();
  pdl_wait();
  const Ep ep = peer_enter(a.sync);
  const int me = a.sync.rank, G = a.sync.world;
  // interleave cycle of G CTAs: CTA k of each cycle serves region (me + 1 + k) % G (k = G - 1: the own region);
  // the launcher sizes the grid in whole cycles
  const int k = (int)(blockIdx.x % G);
  const int64_t local_cta = blockIdx.x / G, n_cta = gridDim.x / G;
  const int64_t tid = local_cta * blockDim.x + threadIdx.x;
  const int64_t stride = n_cta * blockDim.x;
  const int64_t slot_off = (int64_t)a.slot[0] * a.reg_len;
  constexpr int U = kScsU;
  const int r = (me + 1 + k) % G;
  const int64_t lo = min((int64_t)r * a.reg_len, a.P), cnt = min((int64_t)(r + 1) * a.reg_len, a.P) - lo;
  float *dst = a.inbox[r] + slot_off;
  const int64_t n4 = cnt >> 2;
  for (int64_t q0 = tid; q0 < n4; q0 += stride * U) {
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = q0 + u * stride;
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (q < n4 && a.n_src > 0) acc[u] = ld4(a.src[0] + lo + 4 * q);
    }
    for (int j0 = 1; j0 < a.n_src; j0 += kG1) {
      float4 t[kG1][U];
#pragma unroll
      for (int jj = 0; jj < kG1; ++jj)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j0 + jj < a.n_src && q0 + u * stride < n4) t[jj][u] = ld4(a.src[j0 + jj] + lo + 4 * (q0 + u * stride));
#pragma unroll
      for (int jj = 0; jj < kG1; ++jj)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j0 + jj < a.n_src && q0 + u * stride < n4) acc[u] = add4(acc[u], t[jj][u]);  // ascending
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * stride < n4) *reinterpret_cast<float4 *>(dst + 4 * (q0 + u * stride)) = acc[u];
  }
  const int64_t i = 4 * n4 + tid;  // scalar tail of the region
  if (i < cnt) {
    float acc = a.n_src > 0 ? a.src[0][lo + i] : 0.0f;
    for (int j = 1; j < a.n_src; ++j) acc = __fadd_rn(acc, a.src[j][lo + i]);
    dst[i] = acc;
  }
  peer_done(a.sync, ep);
}

// ---------------------------------------------------------------------------------------------------------------
// K3 synth_grad: g = ((h >> 40) * 2^-24 - 0.5) * 2^-6 with h = splitmix64(seed ^ ((j<<56) ^ (k<<30) ^ i)).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float synth1(uint64_t seed, uint64_t jk, uint64_t i) {
  const uint64_t h = splitmix64(seed ^ (jk ^ i));
  const float u = __fmul_rn((float)(uint32_t)(h >> 40), 5.9604644775390625e-08f);  // * 2^-24, exact
  return __fmul_rn(__fadd_rn(u, -0.5f), 0.015625f);                                // exact
}

__global__ void __launch_bounds__(kThreads) synth_grad_kernel(uint64_t seed, uint64_t jk, int64_t i0, int64_t count,
                                                              float *dst, bool vec) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t n4 = count >> 2;
    for (int64_t q = tid; q < n4; q += stride) {
      const uint64_t i = (uint64_t)(i0 + 4 * q);
      st4(dst + 4 * q, make_float4(synth1(seed, jk, i), synth1(seed, jk, i + 1), synth1(seed, jk, i + 2),
                                   synth1(seed, jk, i + 3)));
    }
    done = 4 * n4;
  }
  for (int64_t t = done + tid; t < count; t += stride) dst[t] = synth1(seed, jk, (uint64_t)(i0 + t));
}

// ---------------------------------------------------------------------------------------------------------------
// K4 softmax regression: logits z = x W (W is d x C row-major), p = softmax(z), r = (p - onehot(y)) / B,
// grad = X^T r, loss = mean_b(-log p_{b,y_b}). Two small kernels; fixed summation orders (deterministic).
constexpr int kMaxC = 32;

__global__ void __launch_bounds__(kThreads) softmax_fwd_kernel(const float *X, const int32_t *y, int32_t B,
                                                               int32_t d, int32_t C, const float *W, float *r,
                                                               float *loss_b) {
  const int b = blockIdx.x;
  const float *x = X + (int64_t)b * d;
  float part[kMaxC];
#pragma unroll
  for (int c = 0; c < kMaxC; ++c) part[c] = 0.0f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float xi = x[i];
    const float *wr = W + (int64_t)i * C;
#pragma unroll
    for (int c = 0; c < kMaxC; ++c)
      if (c < C) part[c] = __fmaf_rn(xi, wr[c], part[c]);
  }
  __shared__ float red[kThreads / 32][kMaxC];
  __shared__ float z[kMaxC];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kMaxC; ++c) {
    if (c >= C) break;
    float s = part[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[wid][c] = s;
  }
  __syncthreads();
  if (threadIdx.x < C) {
    float s = 0.0f;
    for (int k = 0; k < kThreads / 32; ++k) s += red[k][threadIdx.x];
    z[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = z[0];
    for (int c = 1; c < C; ++c) m = fmaxf(m, z[c]);
    float den = 0.0f;
    for (int c = 0; c < C; ++c) den += expf(z[c] - m);
    const int yb = y[b];
    loss_b[b] = -((z[yb] - m) - logf(den));
    // r = (p - onehot(y)) / B. For the true class p_y - 1 = -sum_{c != y} p_c: summing the other classes avoids the
    // cancellation of p_y - 1 in fp32 when the model is confident (p_y -> 1).
    float rest = 0.0f;
    for (int c = 0; c < C; ++c) {
      if (c == yb) continue;
      const float p = expf(z[c] - m) / den;
      rest += p;
      r[(int64_t)b * C + c] = p / (float)B;
    }
    r[(int64_t)b * C + yb] = -rest / (float)B;
  }
}

__global__ void __launch_bounds__(kThreads) softmax_bwd_kernel(const float *X, int32_t B, int32_t d, int32_t C,
                                                               const float *r, const float *loss_b, float *grad,
                                                               float *loss) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < (int64_t)d * C) {
    const int64_t i = idx / C;
    const int c = (int)(idx % C);
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s = __fmaf_rn(X[(int64_t)b * d + i], r[(int64_t)b * C + c], s);
    grad[idx] = s;
  }
  if (idx == 0) {
    float s = 0.0f;
    for (int b = 0; b < B; ++b) s += loss_b[b];
    *loss = s / (float)B;
  }
}

// ---------------------------------------------------------------------------------------------------------------
// Dynamic switching criterion for the toy model. With per-sample gradients
// grad_b = x_b (x) (p_b - y_b) (rank one) and the batch mean g, Delta = g - g_prev:
//   u_b = Delta^T (grad_b - g) = x_b^T Delta (p_b - y_b) - Delta^T g,  sigma = sqrt(sum_b u_b^2) / (B |Delta|).
// r = (p - y)/B from softmax_fwd, so x_b^T Delta (p_b - y_b) = B * sum_i x_b[i] sum_c Delta[i,c] r[b,c]. One CTA per
// sample (plus one for |Delta|^2 and Delta^T g), fp64 accumulation in a fixed order; a final 1-CTA kernel.
__global__ void __launch_bounds__(kThreads) criterion_partial_kernel(const float *X, int32_t B, int32_t d, int32_t C,
                                                                     const float *r, const float *g,
                                                                     const float *g_prev, double *part) {
  const int b = blockIdx.x;  // b < B: sample b; b == B: global terms
  double acc0 = 0.0, acc1 = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    if (b < B) {
      double t = 0.0;
      for (int c = 0; c < C; ++c) {
        const int64_t k = (int64_t)i * C + c;
        t += (double)(g[k] - g_prev[k]) * (double)r[(int64_t)b * C + c];
      }
      acc0 += (double)X[(int64_t)b * d + i] * t;
    } else {
      for (int c = 0; c < C; ++c) {
        const int64_t k = (int64_t)i * C + c;
        const double dl = (double)g[k] - (double)g_prev[k];
        acc0 += dl * dl;
        acc1 += dl * (double)g[k];
      }
    }
  }
  __shared__ double red0[kThreads / 32], red1[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    acc0 += __shfl_down_sync(0xffffffffu, acc0, o);
    acc1 += __shfl_down_sync(0xffffffffu, acc1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red0[threadIdx.x >> 5] = acc0;
    red1[threadIdx.x >> 5] = acc1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) {
      s0 += red0[w];
      s1 += red1[w];
    }
    if (b < B) {
      part[b] = s0 * (double)B;        // x_b^T Delta (p_b - y_b)
    } else {
      part[B] = s0;                    // |Delta|^2
      part[B + 1] = s1;                // Delta^T g
    }
  }
}

__global__ void criterion_final_kernel(int32_t B, const double *part, float *stats) {
  if (threadIdx.x != 0) return;
  const double nd2 = part[B], dg = part[B + 1];
  double su = 0.0;
  for (int b = 0; b < B; ++b) {
    const double u = part[b] - dg;
    su += u * u;
  }
  const double nd = sqrt(nd2);
  stats[0] = (float)nd;
  stats[1] = nd > 0.0 ? (float)(sqrt(su) / ((double)B * nd)) : 0.0f;
}

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

// Grid: enough CTAs for the work, capped at (resident CTAs per SM) x (SM count) — one full wave of a persistent
// grid-stride kernel (B200: 148 SMs).
// Resident CTAs per SM, queried once per kernel (a host API call per launch would dominate small launches).
// Keyed by the kernel's address: kernels of the same signature share a function-pointer type.
template <typename K>
int resident_ctas(K kernel) {
  static std::unordered_map<const void *, int> cache;
  static std::mutex mu;                       // contexts may live on different threads
  std::lock_guard<std::mutex> lock(mu);
  const void *key = reinterpret_cast<const void *>(kernel);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int r = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kernel, kThreads, 0);
  if (r <= 0) r = 1;
  cache[key] = r;
  return r;
}

template <typename K>
int grid_for(K kernel, int64_t work_items) {
  const int resident = resident_ctas(kernel);
  int64_t want = (work_items + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)resident * num_sms();
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

}  // namespace

// Launch with programmatic stream serialization (see pdl_trigger / pdl_wait): only kernels that call pdl_wait before
// touching global data written by earlier work are launched this way, and only on one GPU. Kernels of the fused
// multi-GPU exchange (cross-GPU flag barriers) launch with ordinary serialisation: there PDL measured slower
// (config 2 at 2 GPUs: 12.3k vs 14.6k steps/s; config 3: 1,192 vs 1,204; profiles/r02_pdl_ab.txt).
inline bool pdl_for(const PeerSync &p) { return p.world <= 1 && !p.has_wait && p.signal_off == 0; }

template <typename Arg>
cudaError_t launch_pdl(void (*k)(Arg), int64_t grid, size_t smem, cudaStream_t s, const Arg &arg, bool pdl = true) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef SS_NO_PDL
  cfg.numAttrs = 0;   // A/B variant (tools/kernel_sweep.py set "pdl"): ordinary stream serialisation
  (void)pdl;
#else
  cfg.numAttrs = pdl ? 1 : 0;
#endif
  return cudaLaunchKernelEx(&cfg, k, arg);
}

cudaError_t launch_bsp_update(const BspArgs &a, bool vec, cudaStream_t s) {
  if (a.count <= 0 && !a.sync.has_wait && a.sync.signal_off == 0) return cudaSuccess;
  if (vec) {
    auto k = bsp_update_kernel<true>;
    const int64_t n4 = a.count / 4;
    if (n4 < (int64_t)resident_ctas(k) * num_sms() * kThreads * kU1) {
      // less than one wave of the streaming form (small P, e.g. config 2): latency-bound, one float4 per thread
      auto ks = bsp_update_kernel<true, 1, 4>;
      return launch_pdl(ks, grid_for(ks, n4 + 1), 0, s, a, pdl_for(a.sync));
    }
    return launch_pdl(k, grid_for(k, (n4 + kU1 - 1) / kU1 + 1), 0, s, a, pdl_for(a.sync));
  }
  auto k = bsp_update_kernel<false>;
  return launch_pdl(k, grid_for(k, a.count), 0, s, a, pdl_for(a.sync));
}

cudaError_t launch_local_sum(const SumArgs &a, bool vec, cudaStream_t s) {
  if (a.count_pad <= 0) return cudaSuccess;
  if (vec) {
    auto k = local_sum_kernel<true>;
    k<<<grid_for(k, (a.count / 4 + kU1 - 1) / kU1 + 1), kThreads, 0, s>>>(a);
  } else {
    auto k = local_sum_kernel<false>;
    k<<<grid_for(k, a.count_pad), kThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_asp_replay(const AspArgs &a, bool vec, cudaStream_t s) {
  if ((a.count <= 0 || a.n_ev <= 0) && !a.sync.has_wait && a.sync.signal_off == 0) return cudaSuccess;
  if (!vec) {
    auto k = asp_replay_scalar_kernel;
    k<<<grid_for(k, a.count), kThreads, 0, s>>>(a);
    return cudaGetLastError();
  }
  static const int r = [] {    // resident CTAs per SM at the streaming form's shared memory (thread-safe static init)
    int res = 0;
    cudaFuncSetAttribute(asp_replay_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemMax);
    cudaFuncSetAttribute(asp_replay_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmemMax);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res, asp_replay_tma_kernel<true>, kThreads, kTmaSmem);
    return res > 0 ? res : 1;
  }();
  const int64_t nvec = (a.count >> 2) << 2;
  AspArgs b = a;
  b.n_item = 0;                  // gradient sources per tile (the kernel lists them in shared memory)
  for (int e = 0; e < a.n_ev; ++e) b.n_item += a.ev[e].kind == 0 ? 1 : a.ev[e].kind == 2 ? a.ev[e].n_src : 0;
  // Small-launch form: one tile per CTA, every gradient source of it staged at once (no stage reuse, no CTA
  // barrier per item), as many CTAs as fit (up to 4 per SM at 64 registers x 256 threads); tiles are a multiple of
  // 32 floats (128 B). Used when such a tile is no longer than the streaming form's.
  if (b.n_item > 0 && b.n_item <= kMaxStages) {   // (config 2, 1 GPU: 61.6k vs 60.8k steps/s streaming-only)
    for (int per_sm = 4; per_sm >= 1; --per_sm) {
      const int64_t want = (int64_t)per_sm * num_sms();
      const int64_t t = std::max<int64_t>(32, ((nvec + want - 1) / want + 31) / 32 * 32);
      if (t > kTmaTile) break;
      const int64_t smem = (int64_t)b.n_item * t * 4;
      if (smem > kTmaSmemMax || per_sm * (smem + 7 * 1024) > 228 * 1024) continue;   // + static smem + reserve
      b.tile = (int32_t)t;
      b.stages = b.n_item;
      const int64_t grid = std::max<int64_t>(1, (nvec + t - 1) / t);
      return launch_pdl(asp_replay_tma_kernel<false>, grid, (size_t)smem, s, b, pdl_for(b.sync));
    }
  }
  // streaming form: grid-stride over kTmaTile tiles, at most one wave of resident CTAs, a kTmaStages-tile ring
  const int64_t slots = (int64_t)r * num_sms();
  const int64_t tile = kTmaTile;
  const int64_t tiles = (nvec + tile - 1) / tile;
  const int64_t grid = std::max<int64_t>(1, std::min(tiles, slots));
  b.tile = (int32_t)tile;
  b.stages = kTmaStages;
  const int64_t items = (tiles + grid - 1) / grid * b.n_item;   // most gradient tiles any CTA stages
  if (items > kTmaStages) return launch_pdl(asp_replay_tma_kernel<true>, grid, kTmaSmem, s, b, pdl_for(b.sync));
  return launch_pdl(asp_replay_tma_kernel<false>, grid, kTmaSmem, s, b, pdl_for(b.sync));
}

cudaError_t launch_scatter_sum(const ScatterArgs &a, cudaStream_t s) {
  auto k = scatter_sum_kernel;
  const int G = a.sync.world > 0 ? a.sync.world : 1;
  const int grid = (std::max(grid_for(k, (a.P / 4 + kScsU - 1) / kScsU + 1), G) + G - 1) / G * G;   // whole cycles
  return launch_pdl(k, grid, 0, s, a, false);
}

cudaError_t launch_scatter(const ScatterArgs &a, cudaStream_t s) {
  auto k = scatter_kernel;
  const int64_t work = a.n_src > 0 ? (a.P / 4 + 3) / 4 + 1 : 1;
  return launch_pdl(k, grid_for(k, work), 0, s, a, false);
}

cudaError_t launch_synth_grad(uint64_t seed, int32_t j, int64_t k, int64_t i0, int64_t count, float *dst,
                              cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const uint64_t jk = ((uint64_t)(uint32_t)j << 56) ^ ((uint64_t)k << 30);
  const bool vec = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  int64_t items = vec ? count / 4 + 1 : count;
  int64_t want = (items + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)num_sms() * 8;
  synth_grad_kernel<<<(int)(want < cap ? want : cap), kThreads, 0, s>>>(seed, jk, i0, count, dst, vec);
  return cudaGetLastError();
}

cudaError_t launch_dynamic_criterion(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C,
                                     const float *W, const float *g_prev, float *g_out, float *stats, float *scratch,
                                     double *part, cudaStream_t s) {
  float *loss = scratch + (int64_t)B * (C + 1);
  cudaError_t e = launch_softmax_grad(X, y, B, d, C, W, g_out, loss, scratch, s);  // r in scratch[0 .. B*C)
  if (e != cudaSuccess) return e;
  criterion_partial_kernel<<<B + 1, kThreads, 0, s>>>(X, B, d, C, scratch, g_out, g_prev, part);
  criterion_final_kernel<<<1, 32, 0, s>>>(B, part, stats);
  return cudaGetLastError();
}

cudaError_t launch_softmax_grad(const float *X, const int32_t *y, int32_t B, int32_t d, int32_t C, const float *W,
                                float *grad, float *loss, float *scratch, cudaStream_t s) {
  float *r = scratch;
  float *loss_b = scratch + (int64_t)B * C;
  softmax_fwd_kernel<<<B, kThreads, 0, s>>>(X, y, B, d, C, W, r, loss_b);
  const int64_t n = (int64_t)d * C;
  softmax_bwd_kernel<<<(int)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(X, B, d, C, r, loss_b, grad, loss);
  return cudaGetLastError();
}

}  // namespace ss
