// Grid-barrier latency microbenchmark (148 CTAs x 544 threads, as decode_mk):
//   A: one counter, red.release.gpu + ld.acquire.gpu poll (decode_mk today)
//   B: per-CTA flag words (st.release), one warp polls all flags
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bar_bench tools/bar_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void cbar() { asm volatile("bar.sync 1, 512;" ::: "memory"); }

__global__ void bar_a(unsigned* ctr, int iters) {
  if (threadIdx.x >= 512) return;
  unsigned target = 0;
  for (int i = 0; i < iters; ++i) {
    cbar();
    target += gridDim.x;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      unsigned v;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    cbar();
  }
}

__global__ void bar_b(unsigned* flags, int iters) {  // flags[c * 32] (128-B apart)
  if (threadIdx.x >= 512) return;
  const int lane = threadIdx.x & 31;
  for (int i = 1; i <= iters; ++i) {
    cbar();
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"((unsigned)i) : "memory");
    if (threadIdx.x < 32) {
      for (int c = lane; c < (int)gridDim.x; c += 32) {
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + c * 32) : "memory"); } while (v < (unsigned)i);
      }
      __syncwarp();
    }
    cbar();
  }
}

__global__ void bar_c(unsigned* flags, int iters) {  // packed flags: 148 words contiguous
  if (threadIdx.x >= 512) return;
  const int lane = threadIdx.x & 31;
  for (int i = 1; i <= iters; ++i) {
    cbar();
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"((unsigned)i) : "memory");
    if (threadIdx.x < 32) {
      for (int c = lane; c < (int)gridDim.x; c += 32) {
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + c) : "memory"); } while (v < (unsigned)i);
      }
      __syncwarp();
    }
    cbar();
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* buf;
  cudaMalloc(&buf, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(buf, 0, 1 << 20);
      cudaEventRecord(e0);
      void* args[] = {&buf, (void*)&iters};
      void* fn = v == 0 ? (void*)bar_a : v == 1 ? (void*)bar_b : (void*)bar_c;
      cudaLaunchCooperativeKernel(fn, sms, 544, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("variant %c: %.3f us per grid barrier (%s)\n", 'A' + v, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
