// plan.h — host-side shard layout, ASP window cutting and per-window routing plan (§8(e)).
// Shared by the runtime (which executes the plan with NCCL or fused peer stores) and by ss_route_plan (CPU tests).
#pragma once
#include <stdint.h>

#include <vector>

namespace ss {

struct Layout {
  int32_t rank = 0, world = 1, n = 1, S = 1;
  int64_t P = 0, pad = 0, P_pad = 0, reg_len = 0;
  std::vector<int64_t> real_lo, real_hi;  // per rank: unpadded element range of its owner region
  int32_t host(int32_t j) const { return (int32_t)(((int64_t)j * world) / n); }  // worker j's GPU
  int32_t first_hosted(int32_t r) const;
  int32_t n_hosted(int32_t r) const;
  int64_t count(int32_t r) const { return real_hi[r] - real_lo[r]; }
};

// pad = ceil(ceil(P/S)/32)*32, P_pad = S*pad; rank r owns [r*P_pad/world, (r+1)*P_pad/world) (S % world == 0).
Layout make_layout(int64_t P, int32_t S, int32_t n, int32_t rank, int32_t world);

struct RouteOp {
  int32_t phase;   // 0: gradient slice pusher -> owner; 1: snapshot slice owner -> puller
  int32_t op;      // 0 send (fused: posted store), 1 recv
  int32_t peer;
  int32_t event;   // index of the event in its window
  int64_t offset;  // element offset of the slice in the full vector
  int64_t count;
};

// Ops of one window as seen by L.rank, in issue order. data[k] = 1 when pull k moves parameters.
void plan_window(const Layout &L, const int32_t *kind, const int32_t *worker, const uint8_t *data, int32_t n_ev,
                 std::vector<RouteOp> &out);

// True when the window must be flushed before appending (kind, worker): it is full, or (fused) it already holds a
// pull of that worker (one mapped pull buffer per hosted worker).
bool window_cut(const int32_t *kind, const int32_t *worker, int32_t n_in_window, int32_t new_kind, int32_t new_worker,
                int32_t max_window, bool fused);

}  // namespace ss
