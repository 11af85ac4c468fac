// scenario.cpp — online straggler scenario (SURVEY config 4): a discrete-event driver that runs the greedy policy
// on the straggler detector over BSP supersteps and the seeded ASP arrival clock, issuing the
// protocol calls (ss_bsp_step / ss_asp_push / ss_pull / ss_switch) on a context, or a host-only dry run.
// Semantics: include/syncswitch.h (ss_scenario_run) and DESIGN.md reading C23.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "internal.h"
#include "syncswitch.h"

namespace {

uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Gradient ring and pull destinations of the run. Buffers passed to the protocol calls are borrowed until ss_sync
// (an ASP window may still reference them), so the ring is released only after a flush + sync, on every exit path.
struct Buffers {
  ss_ctx *ctx = nullptr;
  std::vector<float *> bsp, asp, pull;
  std::vector<float *> owned;
  ~Buffers() {
    if (ctx) ss_sync(ctx);
    for (float *p : owned) cudaFree(p);
  }
};

}  // namespace

extern "C" ss_status ss_scenario_run(ss_ctx *ctx, const ss_scenario *sc, ss_scenario_result *out,
                                     ss_switch_event *log, int32_t cap) {
  if (!sc || !out || cap < 0 || (cap > 0 && !log)) return SS_E_INVAL;
  const int32_t n = sc->n_workers;
  if (n < 1 || n > ss::kMaxWorkers || sc->batch < 1 || sc->total_samples < 1 || sc->quota_den < 1 ||
      sc->quota_num < 0 || sc->quota_num > sc->quota_den || sc->jitter < 0 || sc->period <= sc->jitter ||
      sc->window_ticks < 1 || sc->K < 1 || sc->slow_factor < 1 || sc->policy < 0 || sc->policy > 2)
    return SS_E_INVAL;

  ss::CtxInfo info{};
  if (ctx) {
    info = ss::ctx_info(ctx);
    if (info.n != n) return SS_E_INVAL;
  }
  auto hosted = [&](int32_t j) { return !ctx || (int32_t)(((int64_t)j * info.world) / n) == info.rank; };

  // device buffers: one BSP gradient per hosted worker, a ring of max_window ASP gradients, a pull destination
  Buffers buf;
  buf.ctx = ctx;
  if (ctx) {
    auto alloc = [&](std::vector<float *> &v, int32_t count) -> bool {
      for (int32_t i = 0; i < count; ++i) {
        float *p = nullptr;
        if (cudaMalloc(&p, (size_t)info.P * sizeof(float)) != cudaSuccess) return false;
        buf.owned.push_back(p);
        v.push_back(p);
      }
      return true;
    };
    if (!alloc(buf.bsp, n) || !alloc(buf.asp, info.max_window)) return SS_E_OOM;
    buf.pull.assign(n, nullptr);
    for (int32_t j = 0; j < n; ++j) {
      if (!hosted(j)) continue;
      if (info.world > 1 && info.fused) {
        if (ss_pull_buffer(ctx, j, &buf.pull[j]) != SS_OK) return SS_E_CUDA;
      } else {
        std::vector<float *> one;
        if (!alloc(one, 1)) return SS_E_OOM;
        buf.pull[j] = one[0];
      }
    }
  }

  const int64_t quota = (int64_t)((__int128)sc->total_samples * sc->quota_num / sc->quota_den);
  const int64_t B = sc->batch, W = sc->total_samples, D = sc->window_ticks;
  std::vector<int64_t> c(n, 0), base(n, 0), dur(n, 0), nxt(n, 0);
  std::vector<double> acc_s(n, 0.0), acc_b(n, 0.0);
  std::vector<int32_t> strag(n, 0);
  int64_t t = 0, done = 0, bsp_done = 0, version = 0, win_end = D, ring = 0;
  int32_t proto = SS_BSP, n_log = 0;
  // BSP barrier set (elastic policy): removed workers stop receiving work until the quota is met
  std::vector<uint8_t> mem(n, 1);
  int32_t n_mem = n;
  ss_scenario_result r{};
  ss_detector *dt = nullptr;
  if (ss_detector_new(&dt, n, sc->K) != SS_OK) return SS_E_INVAL;
  struct Guard {
    ss_detector *d;
    ~Guard() { ss_detector_free(d); }
  } guard{dt};

  auto period = [&](int32_t j, int64_t at) {
    return (j == sc->slow_worker && at >= sc->slow_t0 && at < sc->slow_t1) ? sc->period * sc->slow_factor
                                                                              : sc->period;
  };
  auto gap = [&](int32_t j, int64_t at) {  // duration of worker j's next step (its (c[j]+1)-th gradient)
    int64_t d = 0;
    if (sc->jitter > 0) {
      const uint64_t h = mix64(sc->sched_seed ^ ((uint64_t)(uint32_t)j << 32) ^ (uint64_t)(c[j] + 1));
      d = (int64_t)(h % (uint64_t)(2 * sc->jitter + 1)) - sc->jitter;
    }
    return period(j, at) + d;
  };
  auto gen = [&](int32_t j, float *dst) -> ss_status {  // worker j's c[j]-th gradient
    if (!ctx || !hosted(j)) return SS_OK;
    return ss::launch_synth_grad(sc->grad_seed, j, c[j], 0, info.P, dst, info.stream) == cudaSuccess ? SS_OK
                                                                                                    : SS_E_CUDA;
  };
  auto do_switch = [&](int32_t to, int32_t reason) -> ss_status {
    if (ctx) {
      ss_status s = ss_switch(ctx, to, 0);
      if (s != SS_OK) return s;
    }
    if (n_log < cap) log[n_log] = ss_switch_event{t, version, to, reason, n_mem};
    ++n_log;
    proto = to;
    return SS_OK;
  };
  auto pull = [&](int32_t j) -> ss_status {
    if (ctx) {
      int64_t v = 0;
      ss_status s = ss_pull(ctx, j, hosted(j) ? buf.pull[j] : nullptr, &v);
      if (s != SS_OK) return s;
    }
    base[j] = version;
    return SS_OK;
  };
  auto start_asp = [&]() -> ss_status {
    for (int32_t j = 0; j < n; ++j) {
      ss_status s = pull(j);
      if (s != SS_OK) return s;
      dur[j] = gap(j, t);
      nxt[j] = t + dur[j];
    }
    return SS_OK;
  };

  auto set_members = [&]() -> ss_status {
    if (!ctx) return SS_OK;
    std::vector<int32_t> ids;
    for (int32_t j = 0; j < n; ++j)
      if (mem[j]) ids.push_back(j);
    return ss_set_members(ctx, ids.data(), (int32_t)ids.size());
  };
  auto log_event = [&](int32_t to, int32_t reason) {
    if (n_log < cap) log[n_log] = ss_switch_event{t, version, to, reason, n_mem};
    ++n_log;
  };

  while (done < W) {
    if (proto == SS_BSP) {
      std::vector<const float *> g;
      std::vector<int32_t> ws;
      std::vector<int64_t> vs;
      // one GPU defers a superstep into the pending window: launch it before its gradient buffers are rewritten
      if (ctx) {
        ss_status s = ss::ctx_flush(ctx);
        if (s != SS_OK) return s;
      }
      for (int32_t j = 0; j < n; ++j) {
        if (!mem[j] || !hosted(j)) continue;
        ss_status s = gen(j, ctx ? buf.bsp[j] : nullptr);
        if (s != SS_OK) return s;
        g.push_back(ctx ? buf.bsp[j] : nullptr);
        ws.push_back(j);
        vs.push_back(version);
      }
      if (ctx) {
        ss_status s = ss_bsp_step(ctx, g.data(), ws.data(), vs.data(), (int32_t)g.size());
        if (s != SS_OK) return s;
      }
      int64_t mx = 0;
      for (int32_t j = 0; j < n; ++j) {
        if (!mem[j]) continue;
        const int64_t dj = gap(j, t);
        acc_b[j] += (double)dj;   // busy time excludes the barrier wait (reading C14)
        acc_s[j] += (double)B;
        mx = std::max(mx, dj);
      }
      for (int32_t j = 0; j < n; ++j)
        if (mem[j]) c[j] += 1;
      version += 1;
      t += mx;
      done += (int64_t)n_mem * B;
      bsp_done += (int64_t)n_mem * B;
      r.bsp_steps += 1;
      if (bsp_done >= quota) {  // timing policy: the BSP share is done; restore every worker, ASP for the rest
        if (n_mem < n) {
          std::fill(mem.begin(), mem.end(), 1);
          n_mem = n;
          ss_status s = set_members();
          if (s != SS_OK) return s;
        }
        ss_status s = do_switch(SS_ASP, 0);
        if (s == SS_OK) s = start_asp();
        if (s != SS_OK) return s;
      }
    } else {
      int32_t j = 0;
      for (int32_t q = 1; q < n; ++q)
        if (nxt[q] < nxt[j]) j = q;
      t = nxt[j];
      float *gbuf = ctx ? buf.asp[ring % info.max_window] : nullptr;
      ++ring;
      ss_status s = gen(j, gbuf);
      if (s != SS_OK) return s;
      if (ctx) {
        int64_t st = 0;
        s = ss_asp_push(ctx, j, hosted(j) ? gbuf : nullptr, base[j], &st);
        if (s != SS_OK) return s;
      }
      c[j] += 1;
      version += 1;
      s = pull(j);
      if (s != SS_OK) return s;
      acc_b[j] += (double)dur[j];
      acc_s[j] += (double)B;
      done += B;
      r.asp_pushes += 1;
      dur[j] = gap(j, t);
      nxt[j] = t + dur[j];
    }
    while (t >= win_end) {  // detection windows closed by time t (the current event is counted in the closing one)
      int32_t clean = 0;
      const bool masked = sc->policy == 1 && proto == SS_BSP;
      ss_detector_window_masked(dt, acc_s.data(), acc_b.data(), masked ? mem.data() : nullptr, strag.data(),
                                &clean);
      std::fill(acc_s.begin(), acc_s.end(), 0.0);
      std::fill(acc_b.begin(), acc_b.end(), 0.0);
      win_end += D;
      r.windows += 1;
      int32_t any = 0;
      for (int32_t q = 0; q < n; ++q) any |= strag[q];
      if (sc->policy == 0) {  // greedy
        const int32_t dec = ss_greedy_decision(proto, any, clean, bsp_done, quota);
        if (dec == SS_ASP) {
          ss_status s = do_switch(SS_ASP, 1);
          if (s == SS_OK) s = start_asp();
          if (s != SS_OK) return s;
        } else if (dec == SS_BSP) {
          ss_status s = do_switch(SS_BSP, 2);
          if (s != SS_OK) return s;
          for (int32_t q = 0; q < n; ++q) {  // every worker's in-flight gradient arrives late and is dropped
            if (ctx) {
              int64_t st = 0;
              s = ss_asp_push(ctx, q, hosted(q) ? buf.asp[0] : nullptr, base[q], &st);
              if (s != SS_E_STATE) return s == SS_OK ? SS_E_STATE : s;
            }
            c[q] += 1;
            r.dropped += 1;
          }
        }
      } else if (sc->policy == 1 && proto == SS_BSP && any && bsp_done < quota) {  // elastic
        int32_t keep = 0;
        for (int32_t q = 0; q < n; ++q) keep += mem[q] && !strag[q];
        if (keep >= 1) {  // at least one non-straggler stays
          for (int32_t q = 0; q < n; ++q)
            if (strag[q]) mem[q] = 0;
          n_mem = keep;
          ss_status s = set_members();
          if (s != SS_OK) return s;
          log_event(SS_BSP, 3);
        }
      }
    }
  }
  r.end_tick = t;
  r.version = version;
  r.n_switches = n_log;
  *out = r;
  return SS_OK;
}
