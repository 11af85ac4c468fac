// launch_probe.cu — back-to-back launch cost of a kernel vs the size of its __grid_constant__ parameter struct and
// its grid (the fused kernels pass 2-3.5 KB structs). Prints device microseconds per launch over 2000 launches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 launch_probe.cu -o launch_probe
#include <cuda_runtime.h>

#include <cstdio>

template <int BYTES>
struct Args {
  unsigned char pad[BYTES];
  int *out;
};

template <int BYTES>
__global__ void k(const __grid_constant__ Args<BYTES> a) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && a.pad[0] == 7) *a.out = 1;
}

template <int BYTES>
float run(int grid, cudaStream_t s, int *out) {
  Args<BYTES> a{};
  a.out = out;
  for (int i = 0; i < 100; ++i) k<BYTES><<<grid, 256, 0, s>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 2000; ++i) k<BYTES><<<grid, 256, 0, s>>>(a);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / 2000.f;
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int *out;
  cudaMalloc(&out, 4);
  for (int grid : {148, 296, 592, 1184}) {
    std::printf("grid %5d: params 64 B %.2f us | 1 KB %.2f us | 2 KB %.2f us | 3.5 KB %.2f us per launch\n", grid,
                run<64>(grid, s, out), run<1024>(grid, s, out), run<2048>(grid, s, out), run<3584>(grid, s, out));
  }
  std::printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
