// Streaming-bandwidth microbenchmark for the decode kernel's weight path:
// one CTA per SM streams its contiguous share of a 1 GiB bf16 matrix through
// a TMA + mbarrier ring (producer lane + consumer warps), as decode_mk.cu does.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bw tools/tma_bw.cu -lcuda
//   tools/tma_bw
//
// Variants: box shape (rows x cols), stage count, consumer work (none / the
// real two-row dot product), 1-D bulk copies, and plain register loads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) { while (!mbar_try(b, par)) {} }
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(b)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ float dot8(uint4 w, uint4 x, float acc) {
  const uint32_t* a = &w.x; const uint32_t* b = &x.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    acc = fmaf(__uint_as_float(a[i] << 16), __uint_as_float(b[i] << 16), acc);
    acc = fmaf(__uint_as_float(a[i] & 0xffff0000u), __uint_as_float(b[i] & 0xffff0000u), acc);
  }
  return acc;
}

struct Cfg { int rows, cols, stages, warps, work, mode; };  // mode 0 = 2D TMA, 1 = 1D bulk
// work: 0 none, 1 rows split over warps (all warps on every tile), 2 one warp per tile

__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, const __nv_bfloat16* W, int N, int K,
                              Cfg cfg, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int S = cfg.stages, W_ = cfg.warps;
  const int tile_bytes = cfg.rows * cfg.cols * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], cfg.work == 2 ? 1 : W_); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int kt = K / cfg.cols, nb = N / cfg.rows;
  const long T = (long)nb * kt;
  const long lo = T * blockIdx.x / gridDim.x, hi = T * (blockIdx.x + 1) / gridDim.x;
  uint8_t* xs_raw = sm + (size_t)S * tile_bytes;
  const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(xs_raw);
  if (warp == W_) {
    if (lane == 0) {
      uint32_t n = 0;
      for (long u = lo; u < hi; ++u, ++n) {
        const int slot = n % S;
        mbar_wait(&empty[slot], ((n / S) & 1) ^ 1);
        mbar_expect_tx(&full[slot], tile_bytes);
        const int b = (int)(u / kt), k = (int)(u % kt);
        if (cfg.mode == 0) tma2d(sm + (size_t)slot * tile_bytes, &map, &full[slot], k * cfg.cols, b * cfg.rows);
        else bulk1d(sm + (size_t)slot * tile_bytes, W + (size_t)u * cfg.rows * cfg.cols, tile_bytes, &full[slot]);
      }
    }
    return;
  }
  float a0 = 0.f, a1 = 0.f;
  uint32_t n = 0;
  if (cfg.work == 2) {  // warp w consumes tiles n = w, w + W, ...; empty count = 1 per tile
    n = warp;
    for (long u = lo + warp; u < hi; u += W_, n += W_) {
      const int slot = n % S;
      mbar_wait(&full[slot], (n / S) & 1);
      const uint8_t* t = sm + (size_t)slot * tile_bytes;
      for (int c = lane * 8; c < cfg.cols; c += 256) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xs + c);
#pragma unroll 8
        for (int r = 0; r < cfg.rows; r += 2) {
          const uint4 w0 = *reinterpret_cast<const uint4*>(t + (r * cfg.cols + c) * 2);
          const uint4 w1 = *reinterpret_cast<const uint4*>(t + ((r + 1) * cfg.cols + c) * 2);
          a0 = dot8(w0, xv, a0);
          a1 = dot8(w1, xv, a1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (a0 + a1 == 12345.f) out[0] = a0;
    return;
  }
  for (long u = lo; u < hi; ++u, ++n) {
    const int slot = n % S;
    mbar_wait(&full[slot], (n / S) & 1);
    if (cfg.work) {
      const uint8_t* t = sm + (size_t)slot * tile_bytes;
      const int rows_per_warp = cfg.rows / W_;
      for (int r = 0; r < rows_per_warp; r += 2) {
        for (int c = lane * 8; c < cfg.cols; c += 256) {
          const uint4 w0 = *reinterpret_cast<const uint4*>(t + ((warp * rows_per_warp + r) * cfg.cols + c) * 2);
          const uint4 w1 = *reinterpret_cast<const uint4*>(t + ((warp * rows_per_warp + r + 1) * cfg.cols + c) * 2);
          const uint4 xv = *reinterpret_cast<const uint4*>(xs + c);
          a0 = dot8(w0, xv, a0);
          a1 = dot8(w1, xv, a1);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
  }
  if (a0 + a1 == 12345.f) out[0] = a0;
}

__global__ void reg_kernel(const __nv_bfloat16* W, long elems, float* out) {
  // plain 16-byte loads, 8 in flight per thread
  const long n16 = elems / 8;
  const uint4* p = reinterpret_cast<const uint4*>(W);
  float acc = 0.f;
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const long k = i + j * stride;
      if (k < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(p + k));
      else v[j] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += __uint_as_float(v[j].x) + __uint_as_float(v[j].w);
  }
  if (acc == 12345.f) out[0] = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int N = 65536, K = 8192;  // 1 GiB bf16
  __nv_bfloat16* W;
  float* out;
  CK(cudaMalloc(&W, (size_t)N * K * 2));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(W, 0, (size_t)N * K * 2));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fp;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fp;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)N * K * 2;
  auto timeit = [&](auto&& launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return bytes / (best * 1e-3) / 1e9;
  };
  std::vector<Cfg> cfgs = {
      {32, 256, 12, 16, 1, 0}, {64, 256, 6, 16, 1, 0}, {32, 256, 12, 8, 1, 0}, {128, 256, 3, 16, 1, 0},
      {32, 256, 12, 16, 0, 0},
  };
  if (argc == 7) cfgs = {Cfg{atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5]), atoi(argv[6])}};
  else printf("reg loads: %.0f GB/s\n", timeit([&] { reg_kernel<<<sms * 4, 256>>>(W, (long)N * K, out); }));
  for (const Cfg& c : cfgs) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {(cuuint32_t)c.cols, (cuuint32_t)c.rows};
    cuuint32_t es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, W, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      continue;
    }
    const int smem = c.stages * c.rows * c.cols * 2 + 16384;
    CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const double gbs = timeit([&] { stream_kernel<<<sms, (c.warps + 1) * 32, smem>>>(map, W, N, K, c, out); });
    CK(cudaGetLastError());
    printf("%s box %3dx%3d stages %2d warps %2d work %d: %.0f GB/s\n", c.mode ? "bulk1d" : "tma2d ", c.rows, c.cols,
           c.stages, c.warps, c.work, gbs);
  }
  return 0;
}
