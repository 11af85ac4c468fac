// mc_bench.cu — microbenchmark: NVSwitch multicast stores (multimem.st) vs P2P stores vs local stores, one process
// driving every visible GPU. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 mc_bench.cu -lcuda -o mc_bench
// Prints GB/s of source bytes written per GPU for each variant (all GPUs write concurrently, each its own slice).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    CUresult r_ = (x);                                                               \
    if (r_ != CUDA_SUCCESS) {                                                        \
      const char *s;                                                                 \
      cuGetErrorString(r_, &s);                                                      \
      std::printf("%s failed: %s\n", #x, s);                                         \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

template <int MODE, int U>
__global__ void store_kernel(float *dst0, float *const *peers, int n_peers, size_t n4, float val) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const float4 v = make_float4(val, val, val, val);
  for (size_t q0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q0 < n4; q0 += stride * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t q = q0 + u * stride;
      if (q >= n4) break;
      if (MODE == 0) {  // multicast
        asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst0 + 4 * q), "f"(v.x),
                     "f"(v.y), "f"(v.z), "f"(v.w)
                     : "memory");
      } else if (MODE == 1) {  // P2P to every peer + local
        *reinterpret_cast<float4 *>(dst0 + 4 * q) = v;
        for (int p = 0; p < n_peers; ++p) *reinterpret_cast<float4 *>(peers[p] + 4 * q) = v;
      } else {  // local only
        *reinterpret_cast<float4 *>(dst0 + 4 * q) = v;
      }
    }
  }
}

int main() {
  CK(cuInit(0));
  int n = 0;
  cudaGetDeviceCount(&n);
  const size_t slice = 64ull << 20;  // bytes each GPU writes (its region)
  const size_t total = slice * n;
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
  std::vector<CUdeviceptr> uc(n), mcv(n);
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
    CK(cuMemAddressReserve(&uc[d], size, gran, 0, 0));
    CK(cuMemMap(uc[d], size, 0, mem, 0));
    CK(cuMemSetAccess(uc[d], size, &acc, 1));
    CK(cuMemAddressReserve(&mcv[d], size, gran, 0, 0));
    CK(cuMemMap(mcv[d], size, 0, mc, 0));
    CK(cuMemSetAccess(mcv[d], size, &acc, 1));
  }
  // P2P: plain cudaMalloc buffers with peer access
  std::vector<float *> p2p(n);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    cudaMalloc(&p2p[d], total);
    for (int e = 0; e < n; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
  }
  std::vector<float **> peer_tab(n);
  for (int d = 0; d < n; ++d) {
    std::vector<float *> t;
    for (int e = 0; e < n; ++e)
      if (e != d) t.push_back(p2p[e] + d * (slice / 4));
    cudaSetDevice(d);
    cudaMalloc(&peer_tab[d], sizeof(float *) * (t.size() + 1));
    cudaMemcpy(peer_tab[d], t.data(), sizeof(float *) * t.size(), cudaMemcpyHostToDevice);
  }
  const size_t n4 = slice / 16;
  for (int mode = 0; mode < 3; ++mode) {
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
          const int grid = 148 * grid_mult;
          float *dst = mode == 0 ? (float *)mcv[d] + d * (slice / 4)
                                 : (mode == 1 ? p2p[d] + d * (slice / 4) : (float *)uc[d] + d * (slice / 4));
          if (mode == 0) store_kernel<0, 4><<<grid, 512>>>(dst, peer_tab[d], n - 1, n4, 1.0f);
          if (mode == 1) store_kernel<1, 4><<<grid, 512>>>(dst, peer_tab[d], n - 1, n4, 1.0f);
          if (mode == 2) store_kernel<2, 4><<<grid, 512>>>(dst, peer_tab[d], n - 1, n4, 1.0f);
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
      const char *name[] = {"multicast", "p2p-all", "local"};
      std::printf("%-10s gpus=%d grid=%3dx148 slice=%zu MB: %.1f us  source %.1f GB/s  delivered %.1f GB/s\n",
                  name[mode], n, grid_mult, slice >> 20, worst * 1e3, slice / (worst * 1e-3) / 1e9,
                  (mode == 2 ? 1 : n) * slice / (worst * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaGetLastError();
  std::printf("last error: %s\n", cudaGetErrorString(e));
  return 0;
}
