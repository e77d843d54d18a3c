// L2-hit latency while the other SMs stream HBM: CTA 0 chases pointers through
// a small (L2-resident) buffer with ld.global.cg; CTAs 1.. stream a 1 GiB
// matrix (plain 16-byte loads, `streamers` CTAs, or none).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_lat tools/l2_lat.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void kern(const uint32_t* chain, const uint4* big, long n16, int iters, int streamers,
                     unsigned long long* out, volatile int* stop) {
  if (blockIdx.x == 0) {
    if (threadIdx.x != 0) return;
    // warm the chain
    uint32_t i = 0;
    for (int k = 0; k < 256; ++k) i = __ldcg(chain + i);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int k = 0; k < iters; ++k) i = __ldcg(chain + i);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = (t1 - t0) / iters;
    out[1] = i;
    *stop = 1;
    return;
  }
  if ((int)blockIdx.x > streamers) return;
  float acc = 0.f;
  const long stride = (long)streamers * blockDim.x;
  long pos = (long)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
  while (!*stop) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      long k = (pos + j * stride) % n16;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(big + k));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += __uint_as_float(v[j].x);
    pos += 8 * stride;
  }
  if (acc == 1.2345f) out[2] = 1;
}

int main() {
  const int n = 1 << 16;  // 256 KB chain
  uint32_t* h = new uint32_t[n];
  for (int i = 0; i < n; ++i) h[i] = (uint32_t)((i * 40503u + 977u) % n);  // scattered
  uint32_t* chain;
  uint4* big;
  unsigned long long* out;
  int* stop;
  const long bytes = 1L << 30;
  cudaMalloc(&chain, n * 4);
  cudaMalloc(&big, bytes);
  cudaMalloc(&out, 64);
  cudaMalloc(&stop, 4);
  cudaMemcpy(chain, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(big, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int streams[] = {0, 16, 64, 147};
  for (int s : streams) {
    cudaMemset(stop, 0, 4);
    kern<<<sms, 512>>>(chain, big, bytes / 16, 20000, s, out, stop);
    cudaDeviceSynchronize();
    unsigned long long r[2];
    cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
    printf("streaming CTAs %3d: L2-hit dependent load latency %llu ns\n", s, r[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
