// K6: verify / prefill GEMM on the 5th-generation tensor cores.
//
//   part[s][m][n] = sum_{k in split s} X[m][k] * W[n][k]
//
// Swap-AB for skinny M: the weight tile is the MMA's M side (128 rows, the
// UMMA_M=128 cta_group::1 shape) and the token tile is the MMA's N side
// (NT = 32..256 tokens), so a verify pass of ~80 tokens streams every weight
// byte exactly once per split while the tensor core sees full 128-row tiles.
//
// Per CTA: warp 0 lane 0 = TMA producer (W box 64x128 and X box 64xNT, both
// 128-byte swizzled, one mbarrier with expect_tx per stage), warp 1 lane 0 =
// MMA issuer (4 x tcgen05.mma K=16 per 64-wide k-block, tcgen05.commit frees
// the stage), warp 2 allocates the NT fp32 TMEM columns; afterwards all four
// warps drain TMEM with tcgen05.ld.32x32b (warp w owns TMEM lanes 32w..32w+31
// = weight rows) and write fp32 split partials, 128 B coalesced per token.
#include <cuda.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace sr {

constexpr int kTcThreads = 128;
constexpr int kBK = 64;                 // k-block: 64 bf16 = one 128-B swizzle row
constexpr int kWRows = 128;             // UMMA_M
constexpr int kWStageBytes = kWRows * kBK * 2;  // 16 KB

template <int NT>
__global__ void __launch_bounds__(kTcThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   float* __restrict__ C, int M, int N, int nkb_total, int splits, int stages,
                   __nv_bfloat16* __restrict__ act) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ __align__(8) uint64_t full_bar[8];
  __shared__ __align__(8) uint64_t empty_bar[8];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base_s;

  constexpr int kXStageBytes = NT * kBK * 2;
  constexpr int kStageBytes = kWStageBytes + kXStageBytes;
  // TMEM columns are allocated in powers of two >= 32
  constexpr int kTmemCols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kWRows, m0 = blockIdx.y * NT, split = blockIdx.z;
  const int per = (nkb_total + splits - 1) / splits;
  const int kb0 = split * per;
  const int kb1 = min(nkb_total, kb0 + per);
  const int nkb = kb1 > kb0 ? kb1 - kb0 : 0;

  // 1024-B aligned carve-up of the dynamic smem ring
  const uint32_t raw = smem_u32(smem_dyn);
  uint8_t* base = smem_dyn + ((1024 - (raw & 1023)) & 1023);

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  grid_launch_dependents();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    // Weights do not depend on the previous kernel: the first ring's worth of
    // weight tiles is requested before the programmatic-dependency wait, so
    // it overlaps the predecessor's tail; activations are loaded after it.
    const int pre = nkb < stages ? nkb : stages;
    for (int i = 0; i < pre; ++i) {
      uint8_t* sw = base + (size_t)i * kStageBytes;
      mbar_expect_tx(&full_bar[i], kStageBytes);
      tma_load_2d(sw, &tmW, &full_bar[i], (kb0 + i) * kBK, n0);
    }
    grid_wait();
    for (int i = 0; i < pre; ++i) {
      uint8_t* sx = base + (size_t)i * kStageBytes + kWStageBytes;
      tma_load_2d(sx, &tmX, &full_bar[i], (kb0 + i) * kBK, m0);
    }
    for (int i = pre; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (uint32_t)(i / stages) & 1u;
      mbar_wait(&empty_bar[s], ph ^ 1u);
      uint8_t* sw = base + (size_t)s * kStageBytes;
      uint8_t* sx = sw + kWStageBytes;
      mbar_expect_tx(&full_bar[s], kStageBytes);
      const int k0 = (kb0 + i) * kBK;
      tma_load_2d(sw, &tmW, &full_bar[s], k0, n0);
      tma_load_2d(sx, &tmX, &full_bar[s], k0, m0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    // a ragged last token tile multiplies only its live columns (N % 16 == 0)
    const int rem = M - m0;
    const uint32_t idesc = umma_idesc(rem >= NT ? NT : ((rem + 15) & ~15));
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (uint32_t)(i / stages) & 1u;
      mbar_wait(&full_bar[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sw = smem_u32(base + (size_t)s * kStageBytes);
      const uint32_t sx = sw + kWStageBytes;
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) {
        umma_bf16(tmem, umma_desc_sw128(sw + k * 32), umma_desc_sw128(sx + k * 32), idesc,
                  (i > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(&empty_bar[s]);
    }
    umma_commit(&done_bar);
  }

  // ---------------- epilogue: TMEM -> fp32 partials ----------------
  grid_wait();  // the predecessor may still read the partial buffer
  if (nkb > 0) {
    mbar_wait(&done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = n0 + warp * 32 + lane;  // weight row == TMEM lane
    float* Cs = C + (size_t)split * M * N;
    const int n_live = min(NT, M - m0);
#pragma unroll 1
    for (int j = 0; j < n_live; j += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)j;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
            "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
            "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
            "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
            "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (act != nullptr) {
        // gate/up fused epilogue: warp w holds one 32-row block of the
        // interleaved layout -- lanes 0-15 gate units, lanes 16-31 their up
        const int f = N >> 1;
        const int unit = ((n0 + warp * 32) >> 5) * 16 + (lane & 15);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float g = __uint_as_float(v[c]);
          const float u = __shfl_down_sync(0xffffffffu, g, 16);
          const int m = m0 + j + c;
          if (lane < 16 && m < M && row < N)
            act[(size_t)m * f + unit] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * u);
        }
      } else if (row < N) {
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int m = m0 + j + c;
          if (m < M) Cs[(size_t)m * N + row] = __uint_as_float(v[c]);
        }
      }
    }
  } else {
    // empty split: contribute zeros
    const int row = n0 + warp * 32 + lane;
    float* Cs = C + (size_t)split * M * N;
    if (row < N)
      for (int c = 0; c < NT; ++c)
        if (m0 + c < M) Cs[(size_t)(m0 + c) * N + row] = 0.f;
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}


// Persistent variant: a CTA walks work items (weight tile, token tile, split)
// w = blockIdx.x, += gridDim.x, with two TMEM accumulators.  Warp 0 streams
// TMA tiles across item boundaries, warp 1 issues the MMAs of item i into
// accumulator i & 1, and warps 2-5 (TMEM lane quadrants 2,3,0,1) drain
// accumulator (i-1) & 1 meanwhile -- the epilogue overlaps the next item's
// main loop instead of idling the tensor core, and CTA setup is paid once.
constexpr int kPsThreads = 192;

template <int NT>
__global__ void __launch_bounds__(kPsThreads, 1)
    gemm_tc_persistent(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                       float* __restrict__ C, int M, int N, int nkb_total, int splits, int stages,
                       __nv_bfloat16* __restrict__ act, int n_tiles_n, int n_tiles_m) {
  extern __shared__ uint8_t smem_dyn[];
  __shared__ __align__(8) uint64_t full_bar[8];
  __shared__ __align__(8) uint64_t empty_bar[8];
  __shared__ __align__(8) uint64_t tfull[2];
  __shared__ __align__(8) uint64_t tempty[2];
  __shared__ uint32_t tmem_base_s;

  constexpr int kXStageBytes = NT * kBK * 2;
  constexpr int kStageBytes = kWStageBytes + kXStageBytes;
  constexpr int kAccCols = NT <= 32 ? 32 : NT <= 64 ? 64 : NT <= 128 ? 128 : 256;
  constexpr int kTmemCols = 2 * kAccCols;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = n_tiles_n * n_tiles_m * splits;
  const int per = (nkb_total + splits - 1) / splits;

  const uint32_t raw = smem_u32(smem_dyn);
  uint8_t* base = smem_dyn + ((1024 - (raw & 1023)) & 1023);

  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  grid_launch_dependents();

  auto item_coords = [&](int w, int& n0, int& m0, int& kb0, int& nkb) {
    const int sp = w % splits;
    const int t = w / splits;
    // token tiles fastest: the CTAs running at the same time share weight
    // tiles, so each weight tile is read from HBM once (not once per token tile)
    m0 = (t % n_tiles_m) * NT;
    n0 = (t / n_tiles_m) * kWRows;
    kb0 = sp * per;
    const int kb1 = min(nkb_total, kb0 + per);
    nkb = kb1 > kb0 ? kb1 - kb0 : 0;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      int it = 0;      // global k-block counter (ring position)
      bool waited = false;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        int n0, m0, kb0, nkb;
        item_coords(w, n0, m0, kb0, nkb);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % stages;
          const uint32_t ph = (uint32_t)(it / stages) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          uint8_t* sw = base + (size_t)s * kStageBytes;
          mbar_expect_tx(&full_bar[s], kStageBytes);
          tma_load_2d(sw, &tmW, &full_bar[s], (kb0 + i) * kBK, n0);
          if (!waited) {  // weights first; activations after the dependency wait
            grid_wait();
            waited = true;
          }
          tma_load_2d(sw + kWStageBytes, &tmX, &full_bar[s], (kb0 + i) * kBK, m0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      int it = 0, j = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x, ++j) {
        int n0, m0, kb0, nkb;
        item_coords(w, n0, m0, kb0, nkb);
        const int b = j & 1;
        // a ragged last token tile multiplies only its live columns (N % 16 == 0)
        const int rem = M - m0;
        const uint32_t idesc = umma_idesc(rem >= NT ? NT : ((rem + 15) & ~15));
        mbar_wait(&tempty[b], (((uint32_t)j >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + (uint32_t)(b * kAccCols);
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % stages;
          const uint32_t ph = (uint32_t)(it / stages) & 1u;
          mbar_wait(&full_bar[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sw = smem_u32(base + (size_t)s * kStageBytes);
          const uint32_t sx = sw + kWStageBytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16(acc, umma_desc_sw128(sw + k * 32), umma_desc_sw128(sx + k * 32), idesc,
                      (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty_bar[s]);
        }
        umma_commit(&tfull[b]);
      }
    }
  } else {  // ---------------- epilogue warps 2..5 ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    bool waited = false;
    int j = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++j) {
      int n0, m0, kb0, nkb;
      item_coords(w, n0, m0, kb0, nkb);
      const int b = j & 1;
      mbar_wait(&tfull[b], ((uint32_t)j >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (!waited) {  // the predecessor may still read the output buffer
        grid_wait();
        waited = true;
      }
      const int split = w % splits;
      const int row = n0 + q * 32 + lane;
      float* Cs = C + (size_t)split * M * N;
      const int n_live = min(NT, M - m0);
#pragma unroll 1
      for (int jj = 0; jj < n_live; jj += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kAccCols + jj);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (nkb == 0) {  // empty split: contributes zeros (the accumulator is stale)
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0u;
        }
        if (act != nullptr) {
          const int f = N >> 1;
          const int unit = ((n0 + q * 32) >> 5) * 16 + (lane & 15);
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float g = __uint_as_float(v[c]);
            const float u = __shfl_down_sync(0xffffffffu, g, 16);
            const int m = m0 + jj + c;
            if (lane < 16 && m < M && row < N)
              act[(size_t)m * f + unit] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * u);
          }
        } else if (row < N) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int m = m0 + jj + c;
            if (m < M) Cs[(size_t)m * N + row] = __uint_as_float(v[c]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------ host ---
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2-D bf16 row-major [rows, cols] tensor map with a (box_cols x box_rows) box,
// 128-B swizzled (the GEMM's K-major operand tiles) or plain row-major
int make_tmap_bf16_box(void* out_map, const void* ptr, int rows, int cols, int box_cols,
                       int box_rows, bool swizzle128) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn((CUtensorMap*)out_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr),
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

int make_tmap_bf16(void* out_map, const void* ptr, int rows, int cols, int box_rows) {
  return make_tmap_bf16_box(out_map, ptr, rows, cols, kBK, box_rows, true);
}

int tc_token_tile(int M) {
  static const int cap = [] {
    const char* e = getenv("SR_GEMM_NT_MAX");  // tuning knob: largest token tile
    const int v = e ? atoi(e) : 128;
    return v == 32 || v == 64 || v == 96 || v == 256 ? v : 128;
  }();
  // 128 is the default cap: at M = 256..1024 the 128 x 128 tiles (3-stage
  // ring, two CTAs per SM) beat 128 x 256 by 5-8 % end to end (7B verify
  // 11.65 -> 10.5 ms at M = 640; SR_GEMM_NT_MAX=256 restores the wide tile)
  // 96: verify passes (~60-100 tokens) would waste a third of a 128 tile's
  // activation traffic and MMA work
  int t = M <= 32 ? 32 : M <= 64 ? 64 : M <= 96 ? 96 : M <= 128 ? 128 : 256;
  return t < cap ? t : cap;
}

// narrow-N GEMMs (O, down: N = d) with long token runs: 256-token tiles would
// leave most SMs idle (7B at M = 640: 84 tiles for 148 SMs); 128-token tiles
// double the tile count and run two CTAs per SM
int tc_pick_tile(int M, int N, int num_sms) {
  int nt = tc_token_tile(M);
  if (nt == 256 && (long)((N + kWRows - 1) / kWRows) * ((M + 255) / 256) < num_sms) nt = 128;
  return nt;
}

int tc_pick_splits(int M, int N, int K, int num_sms, int nt_in) {
  const int nt = nt_in ? nt_in : tc_token_tile(M);
  const int tiles = ((N + kWRows - 1) / kWRows) * ((M + nt - 1) / nt);
  const int nkb = K / kBK;
  // token tiles <= 128 run a 3-stage ring, two CTAs per SM: fill both slots
  static const int per_sm = [] {
    const char* e = getenv("SR_GEMM_CTAS_PER_SM");
    const int v = e ? atoi(e) : 2;
    return v < 1 ? 1 : v > 2 ? 2 : v;
  }();
  int s = (nt <= 128 ? per_sm : 1) * num_sms / tiles;
  if (s < 1) s = 1;
  if (s > 8) s = 8;
  while (s > 1 && nkb / s < 4) --s;
  return s;
}

static int gemm_persistent_mode() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_GEMM_PERSIST");
    v = e ? atoi(e) : 2;  // always persistent: 1-3 % faster than per-tile CTAs at M = 80..1024
  }
  return v;
}

template <int NT>
static cudaError_t launch_persistent(const TcGemmArgs& a, cudaStream_t stream, int num_sms) {
  constexpr int stage_bytes = kWStageBytes + NT * kBK * 2;
  // NT <= 128: two CTAs per SM (2 x 2*128 TMEM columns, ~100 KB ring each)
  const int per_sm = NT <= 128 ? 2 : 1;
  int stages = (NT <= 128 ? 100 * 1024 : 200 * 1024) / stage_bytes;
  if (stages > 8) stages = 8;
  const int smem = stages * stage_bytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_persistent<NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tn = (a.N + kWRows - 1) / kWRows, tm = (a.M + NT - 1) / NT;
  const int items = tn * tm * a.splits;
  int grid = per_sm * num_sms;
  if (grid > items) grid = items;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPsThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_tc_persistent<NT>, *(const CUtensorMap*)a.tmW,
                            *(const CUtensorMap*)a.tmX, a.C, a.M, a.N, a.K / kBK, a.splits, stages,
                            a.splits == 1 ? a.act : nullptr, tn, tm);
}

template <int NT>
static cudaError_t launch_nt(const TcGemmArgs& a, cudaStream_t stream) {
  // persistent when the work exceeds one wave of CTA slots (batched verify,
  // long prefill chunks, the 32B gate/up): no wave quantisation, and the
  // TMEM drain overlaps the next tile; one-wave grids keep the plain kernel
  // (measured equal or slightly faster at M ~ 80 for 1.5B / 7B)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int mode = gemm_persistent_mode();  // 1 auto, 2 always, 0 never
  const long items = (long)((a.N + kWRows - 1) / kWRows) * ((a.M + NT - 1) / NT) * a.splits;
  const long slots = (long)(NT <= 128 ? 2 : 1) * sms;
  if (mode == 2 || (mode == 1 && items > slots)) return launch_persistent<NT>(a, stream, sms);
  constexpr int stage_bytes = kWStageBytes + NT * kBK * 2;
  static const int max_stages = [] {
    const char* e = getenv("SR_GEMM_STAGES");  // tuning knob (smaller: 2 CTAs per SM)
    const int v = e ? atoi(e) : 8;
    return v < 2 ? 2 : v > 8 ? 8 : v;
  }();
  int stages = (200 * 1024) / stage_bytes;
  if (stages > max_stages) stages = max_stages;
  // verify-sized token tiles: a 3-deep ring fits two CTAs per SM, so one
  // CTA's TMEM drain overlaps the other's main loop (measured ~4 % at M = 80)
  if (NT <= 128 && max_stages == 8) stages = 3;
  const int smem = stages * stage_bytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((a.N + kWRows - 1) / kWRows, (a.M + NT - 1) / NT, a.splits);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<NT>, *(const CUtensorMap*)a.tmW,
                            *(const CUtensorMap*)a.tmX, a.C, a.M, a.N, a.K / kBK, a.splits, stages,
                            a.splits == 1 ? a.act : nullptr);
}

cudaError_t gemm_tc_launch(const TcGemmArgs& a, cudaStream_t stream) {
  if (a.K % kBK != 0) return cudaErrorInvalidValue;
  switch (a.nt ? a.nt : tc_token_tile(a.M)) {
    case 32: return launch_nt<32>(a, stream);
    case 64: return launch_nt<64>(a, stream);
    case 96: return launch_nt<96>(a, stream);
    case 128: return launch_nt<128>(a, stream);
    default: return launch_nt<256>(a, stream);
  }
}

}  // namespace sr
