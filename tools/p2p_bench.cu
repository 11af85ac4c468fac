// p2p_bench.cu — microbenchmark of all-to-all NVLink writes (the fused path's scatter / pull pattern): every GPU
// sends `bytes` from its own HBM to each peer at the same time, through
//   sm-st   per-thread 16-byte loads + stores (U in flight per thread), the form the fused kernels use;
//   tma     1-D cp.async.bulk tiles HBM -> shared memory, then cp.async.bulk shared -> peer memory;
//   ce      cudaMemcpyPeerAsync on one stream per destination (copy engines).
// One process drives every visible GPU. Prints GB/s sent per GPU (sum over its peers) for each variant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 p2p_bench.cu -o p2p_bench
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));    \
      return 1;                                                                         \
    }                                                                                   \
  } while (0)

constexpr int kMaxPeers = 8;
struct Dst {
  float *p[kMaxPeers];
  int n;
};

// destination order rotated per source GPU (me+1, me+2, ...), one contiguous segment per destination
template <int U>
__global__ void sm_store(const float *src, Dst d, size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int k = 0; k < d.n; ++k) {
    float *dst = d.p[k];
    for (size_t q0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q0 < n4; q0 += stride * U) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < n4) x[u] = __ldcs(reinterpret_cast<const float4 *>(src) + q0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < n4) reinterpret_cast<float4 *>(dst)[q0 + u * stride] = x[u];
    }
  }
}

// interleaved destinations: CTA b serves destination b % n (all links busy from the start)
template <int U>
__global__ void sm_store_split(const float *src, Dst d, size_t n4) {
  const int k = blockIdx.x % d.n;
  const size_t n_cta = (gridDim.x - k + d.n - 1) / d.n;
  const size_t stride = n_cta * blockDim.x;
  float *dst = d.p[k];
  for (size_t q0 = (blockIdx.x / d.n) * (size_t)blockDim.x + threadIdx.x; q0 < n4; q0 += stride * U) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * stride < n4) x[u] = __ldcs(reinterpret_cast<const float4 *>(src) + q0 + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q0 + u * stride < n4) reinterpret_cast<float4 *>(dst)[q0 + u * stride] = x[u];
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// TMA: tiles of TILE bytes, STAGES buffers per CTA; thread 0 issues load (mbarrier) then bulk store (bulk group)
template <int TILE, int STAGES>
__global__ void tma_copy(const float *src, Dst d, size_t bytes) {
  extern __shared__ __align__(128) unsigned char buf[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t tiles = (bytes + TILE - 1) / TILE;
  uint32_t phase[STAGES] = {};
  int it = 0;
  for (int k = 0; k < d.n; ++k) {
    const int kk = (k + blockIdx.x) % d.n;
    for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int s = it % STAGES;
      const size_t off = t * TILE;
      const uint32_t len = (uint32_t)((bytes - off) < TILE ? (bytes - off) : TILE);
      // buffer s is reusable once its previous bulk store has read shared memory
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(len)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(buf + (size_t)s * TILE)),
          "l"((const char *)src + off), "r"(len), "r"(smem_u32(&bar[s]))
          : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(&bar[s])), "r"(phase[s])
            : "memory");
      phase[s] ^= 1;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char *)d.p[kk] + off),
                   "r"(smem_u32(buf + (size_t)s * TILE)), "r"(len)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (G < 2) {
    std::printf("needs >= 2 GPUs\n");
    return 0;
  }
  const size_t bytes = (argc > 1 ? std::atoll(argv[1]) : 64) << 20;   // per destination
  std::vector<float *> src(G);
  std::vector<std::vector<float *>> inbox(G, std::vector<float *>(G, nullptr));   // inbox[dst][src]
  std::vector<cudaStream_t> st(G);
  std::vector<std::vector<cudaStream_t>> ce(G, std::vector<cudaStream_t>(G));
  int sms = 0;
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < G; ++p)
      if (p != g) CK(cudaDeviceEnablePeerAccess(p, 0));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMemset(src[g], 1, bytes));
    for (int s = 0; s < G; ++s)
      if (s != g) CK(cudaMalloc(&inbox[g][s], bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    for (int p = 0; p < G; ++p) CK(cudaStreamCreateWithFlags(&ce[g][p], cudaStreamNonBlocking));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g);
  }
  auto dsts = [&](int g) {
    Dst d{};
    for (int k = 1; k < G; ++k) d.p[d.n++] = inbox[(g + k) % G][g];
    return d;
  };
  auto time_it = [&](const char *name, auto launch) -> int {
    for (int rep = 0; rep < 2; ++rep) {   // warm-up
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        launch(g);
      }
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        cudaDeviceSynchronize();
      }
    }
    const int iters = 10;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) {
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        launch(g);
      }
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        cudaDeviceSynchronize();
      }
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
    CK(cudaGetLastError());
    std::printf("%-28s gpus=%d  %7.1f us  %6.1f GB/s sent per GPU (%d peers x %zu MB)\n", name, G, s * 1e6,
                (double)bytes * (G - 1) / s / 1e9, G - 1, bytes >> 20);
    return 0;
  };
  const size_t n4 = bytes / 16;
  for (int mult : {1, 2, 4}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "sm-st U=8 grid=%dx%d", mult, sms);
    time_it(nm, [&](int g) { sm_store<8><<<mult * sms, 256, 0, st[g]>>>(src[g], dsts(g), n4); });
    std::snprintf(nm, sizeof nm, "sm-st-split U=4 grid=%dx%d", mult, sms);
    time_it(nm, [&](int g) { sm_store_split<4><<<mult * sms, 256, 0, st[g]>>>(src[g], dsts(g), n4); });
  }
  {
    constexpr int T = 16384, S = 4;
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      cudaFuncSetAttribute(tma_copy<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, T * S);
    }
    for (int mult : {1, 2, 4}) {
      char nm[64];
      std::snprintf(nm, sizeof nm, "tma 16KBx4 grid=%dx%d", mult, sms);
      time_it(nm, [&](int g) { tma_copy<T, S><<<mult * sms, 32, T * S, st[g]>>>(src[g], dsts(g), bytes); });
    }
  }
  {
    constexpr int T = 32768, S = 6;
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      cudaFuncSetAttribute(tma_copy<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, T * S);
    }
    time_it("tma 32KBx6 grid=1x148", [&](int g) {
      tma_copy<T, S><<<sms, 32, T * S, st[g]>>>(src[g], dsts(g), bytes);
    });
  }
  time_it("ce memcpyPeer per dest", [&](int g) {
    for (int k = 1; k < G; ++k) {
      const int p = (g + k) % G;
      cudaMemcpyPeerAsync(inbox[p][g], p, src[g], g, bytes, ce[g][p]);
    }
  });
  std::printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
