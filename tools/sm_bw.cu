// Per-SM streaming rate under full-GPU load: every CTA (one per SM) reads an
// equal contiguous slice of a buffer larger than L2 and records its elapsed
// time and %smid.  Run with the slice assignment rotated by R CTAs to tell
// "this SM is slow" (pattern follows smid) from "this address range is slow"
// (pattern follows the slice).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sm_bw tools/sm_bw.cu
//   tools/sm_bw [rotate]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(512, 1) stream(const uint4* buf, size_t per_cta, int rot,
                                                 unsigned long long* t_out, unsigned* sm_out,
                                                 unsigned* sink) {
  __shared__ unsigned long long t0;
  const int slice = (blockIdx.x + rot) % gridDim.x;
  const uint4* p = buf + (size_t)slice * per_cta;
  // grid-wide start: spin until every CTA has arrived
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(sink + 1, 1u);
    while (atomicAdd(sink + 1, 0u) < gridDim.x) {}
    t0 = gns();
  }
  __syncthreads();
  unsigned acc = 0;
  for (size_t i = threadIdx.x; i < per_cta; i += 8 * blockDim.x) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t j = i + (size_t)u * blockDim.x;
      v[u] = j < per_cta ? __ldcs(p + j) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, acc);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    t_out[blockIdx.x] = gns() - t0;
    sm_out[blockIdx.x] = s;
  }
}

int main(int argc, char** argv) {
  int rot = argc > 1 ? atoi(argv[1]) : 0;
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const size_t bytes = (size_t)1 << 30;
  const size_t per = bytes / 16 / nsm;
  uint4* buf;
  unsigned long long* t;
  unsigned *sm, *sink;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaMalloc(&t, nsm * 8);
  cudaMalloc(&sm, nsm * 4);
  cudaMalloc(&sink, 8);
  std::vector<double> acc(nsm, 0.0);
  std::vector<unsigned> smid(nsm);
  const int reps = 5;
  for (int r = 0; r < reps + 1; ++r) {
    cudaMemset(sink, 0, 8);
    stream<<<nsm, 512>>>(buf, per, rot, t, sm, sink);
    std::vector<unsigned long long> ht(nsm);
    cudaMemcpy(ht.data(), t, nsm * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(smid.data(), sm, nsm * 4, cudaMemcpyDeviceToHost);
    if (r == 0) continue;  // warm-up
    for (int i = 0; i < nsm; ++i) acc[smid[i]] += ht[i] / 1e3 / reps;  // us, indexed by smid
  }
  if (cudaError_t e = cudaGetLastError()) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; }
  printf("{\"rotate\": %d, \"bytes_per_cta\": %zu, \"us_by_smid\": [", rot, per * 16);
  for (int i = 0; i < nsm; ++i) printf("%s%.2f", i ? ", " : "", acc[i]);
  printf("]}\n");
  return 0;
}
