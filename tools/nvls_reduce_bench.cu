// nvls_reduce_bench.cu — microbenchmark of the two owner-kernel forms of the multi-GPU BSP exchange (SURVEY §8(f)
// NEXT-1), one process driving every visible GPU, every GPU owning one region of `region` bytes:
//   p2p-pull      owner loads its region of every GPU's gradient (local + NVLink loads), sums, stores locally
//   p2p-pull+bc   ... and stores the sum into every peer's replica (P2P stores): the pull-based one-kernel exchange
//   nvls-ldr      owner reads its region through the multicast view with multimem.ld_reduce (the switch sums the G
//                 copies), stores locally
//   nvls-ldr+st   ... and writes the result with multimem.st into every replica: the NVLS one-kernel exchange
// Reports the time of the slowest GPU and the bus bandwidth in the NCCL convention 2(G-1)/G * (G * region) / t.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 nvls_reduce_bench.cu -lcuda -o nvls_reduce_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                \
  do {                                                       \
    CUresult r_ = (x);                                       \
    if (r_ != CUDA_SUCCESS) {                                \
      const char *s;                                         \
      cuGetErrorString(r_, &s);                              \
      std::printf("%s failed: %s\n", #x, s);                 \
      return 1;                                              \
    }                                                        \
  } while (0)

constexpr int kMaxG = 8;
struct Srcs {
  const float *p[kMaxG];   // every GPU's gradient region (this GPU's own first)
  float *bc[kMaxG];        // peers' replica regions
};

__device__ __forceinline__ float4 ldr4(const float *p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mst4(float *p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

template <int MODE, int U>
__global__ void __launch_bounds__(512) owner_kernel(Srcs s, int G, float *mc_src, float *mc_dst, float *dst,
                                                    size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t q0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q0 < n4; q0 += stride * U) {
    float4 acc[U];
    if (MODE <= 1) {
      float4 t[kMaxG][U];
#pragma unroll
      for (int e = 0; e < kMaxG; ++e)
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (e < G && q0 + u * stride < n4)
            t[e][u] = __ldcg(reinterpret_cast<const float4 *>(s.p[e]) + q0 + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u] = t[0][u];
#pragma unroll
        for (int e = 1; e < kMaxG; ++e)
          if (e < G) acc[u] = make_float4(acc[u].x + t[e][u].x, acc[u].y + t[e][u].y, acc[u].z + t[e][u].z,
                                          acc[u].w + t[e][u].w);
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (q0 + u * stride < n4) acc[u] = ldr4(mc_src + 4 * (q0 + u * stride));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t q = q0 + u * stride;
      if (q >= n4) continue;
      if (MODE == 3) {
        mst4(mc_dst + 4 * q, acc[u]);
      } else {
        reinterpret_cast<float4 *>(dst)[q] = acc[u];
        if (MODE == 1)
          for (int e = 1; e < G; ++e) reinterpret_cast<float4 *>(s.bc[e])[q] = acc[u];
      }
    }
  }
}

struct Mc {
  std::vector<CUdeviceptr> uc, mcv;
};

static int make_mc(int n, size_t total, Mc *out) {
  CUmulticastObjectProp prop{};
  prop.numDevices = n;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  prop.size = total;
  size_t gran;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (total + gran - 1) / gran * gran;
  prop.size = size;
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &prop));
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    CK(cuMulticastAddDevice(mc, dev));
  }
  out->uc.resize(n);
  out->mcv.resize(n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaFree(0);
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemAddressReserve(&out->uc[d], size, gran, 0, 0));
    CK(cuMemMap(out->uc[d], size, 0, mem, 0));
    CK(cuMemSetAccess(out->uc[d], size, &acc, 1));
    CK(cuMemAddressReserve(&out->mcv[d], size, gran, 0, 0));
    CK(cuMemMap(out->mcv[d], size, 0, mc, 0));
    CK(cuMemSetAccess(out->mcv[d], size, &acc, 1));
  }
  return 0;
}

int main(int argc, char **argv) {
  CK(cuInit(0));
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n > kMaxG) n = kMaxG;
  const size_t region = (argc > 1 ? (size_t)atoll(argv[1]) : 32ull) << 20;   // MB owned per GPU
  const size_t total = region * n;
  Mc src, dst;
  if (make_mc(n, total, &src) || make_mc(n, total, &dst)) return 1;
  std::vector<float *> g(n), w(n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaMalloc(&g[d], total);
    cudaMalloc(&w[d], total);
    cudaMemset(g[d], 0, total);
    cudaMemset((void *)src.uc[d], 0, total);
    for (int e = 0; e < n; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
  }
  const size_t n4 = region / 16, rf = region / 4;
  const char *name[] = {"p2p-pull", "p2p-pull+bc", "nvls-ldr", "nvls-ldr+st"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid_mult : {1, 2, 4}) {
      std::vector<cudaEvent_t> a(n), b(n);
      for (int rep = 0; rep < 6; ++rep) {
        for (int d = 0; d < n; ++d) {
          cudaSetDevice(d);
          if (rep == 5) {
            cudaEventCreate(&a[d]);
            cudaEventCreate(&b[d]);
            cudaEventRecord(a[d]);
          }
          Srcs s{};
          for (int k = 0; k < n; ++k) {
            const int e = (d + k) % n;   // own region first, then the peers in rotated order
            s.p[k] = g[e] + d * rf;
            s.bc[k] = w[e] + d * rf;
          }
          float *mcs = (float *)src.mcv[d] + d * rf, *mcd = (float *)dst.mcv[d] + d * rf;
          float *dl = (mode >= 2 ? (float *)dst.uc[d] : w[d]) + d * rf;
          const int grid = 148 * grid_mult;
          if (mode == 0) owner_kernel<0, 2><<<grid, 512>>>(s, n, mcs, mcd, dl, n4);
          if (mode == 1) owner_kernel<1, 2><<<grid, 512>>>(s, n, mcs, mcd, dl, n4);
          if (mode == 2) owner_kernel<2, 4><<<grid, 512>>>(s, n, mcs, mcd, dl, n4);
          if (mode == 3) owner_kernel<3, 4><<<grid, 512>>>(s, n, mcs, mcd, dl, n4);
          if (rep == 5) cudaEventRecord(b[d]);
        }
        for (int d = 0; d < n; ++d) {
          cudaSetDevice(d);
          cudaDeviceSynchronize();
        }
      }
      float worst = 0;
      for (int d = 0; d < n; ++d) {
        float ms;
        cudaSetDevice(d);
        cudaEventElapsedTime(&ms, a[d], b[d]);
        if (ms > worst) worst = ms;
      }
      const double t = worst * 1e-3;
      const double busbw = 2.0 * (n - 1) / n * (double)total / t / 1e9;   // as one RS + AG of the whole vector
      std::printf("%-12s gpus=%d grid=%dx148 region=%zu MB: %8.1f us   busbw(RS+AG) %7.1f GB/s  (%5.1f%% of 900)\n",
                  name[mode], n, grid_mult, region >> 20, worst * 1e3, busbw, busbw / 9.0);
    }
  }
  cudaError_t e = cudaGetLastError();
  std::printf("last error: %s\n", cudaGetErrorString(e));
  return 0;
}
