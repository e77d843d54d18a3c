// Decode-path GEMVs (batch-1 token): HBM-bound weight streaming with fused
// prologues (RMSNorm, embedding gather) and epilogues (bias + RoPE + K/V page
// append, residual add, SiLU*up, greedy argmax + stop test).
//
// Layout: W is row-major [N, K] bf16 (out_features x in_features).  A CTA of
// 8 warps stages the input vector x (bf16, K elements) in shared memory; every
// warp owns a "task" of ROWS rows and streams them with 16-byte
// ld.global.nc.L1::no_allocate loads, U chunks of 256 elements in flight per
// row, fp32 accumulation and a warp-shuffle reduction.  Grids are at most one
// wave (grid-stride over tasks) so that programmatic dependent launch can start
// the next kernel's weight prefetch on the free slots while this one drains.
#include "common.cuh"
#include "kernels.h"

namespace sr {

enum { IN_X = 0, IN_H_NORM = 1, IN_EMBED_NORM = 2 };
enum { EPI_QKV = 0, EPI_RESID = 1, EPI_GLU = 2, EPI_ARGMAX = 3, EPI_LOGITS = 4 };

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;
constexpr int kChunk = 256;  // elements per warp-wide 16-byte load

template <int ROWS>
SR_DEV void task_rows(int epi, int task, const GemvParams& p, int (&r)[ROWS]) {
  if constexpr (ROWS == 2) {
    if (epi == EPI_QKV) {
      const int qk_pairs = (p.q_dim + p.kv_dim) / 2;
      if (task < qk_pairs) {            // rotate-half partners (j, j + 64) of one head
        const int head = task / kHalf, j = task % kHalf;
        r[0] = head * kHeadDim + j;
        r[1] = r[0] + kHalf;
      } else {                          // v rows: any pair
        r[0] = p.q_dim + p.kv_dim + 2 * (task - qk_pairs);
        r[1] = r[0] + 1;
      }
    } else if (epi == EPI_GLU) {        // gate row / up row of one ffn unit
      const int b = task >> 4, j = task & 15;
      r[0] = 32 * b + j;
      r[1] = r[0] + 16;
    } else {
      r[0] = 2 * task;
      r[1] = 2 * task + 1;
    }
  } else {
    r[0] = task;
  }
}

template <int IN, int EPI, int ROWS, int U>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(GemvParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __shared__ float red[32];
  __shared__ float s_v1[kGemvWarps], s_v2[kGemvWarps];
  __shared__ int s_i1[kGemvWarps];
  __shared__ bool s_last;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = p.K;
  const int n_tasks = p.n_tasks;
  const int stride = gridDim.x * kGemvWarps;
  const int nchunk = (K + kChunk - 1) / kChunk;

  // ---- weight prefetch of the first task (independent of predecessors) ----
  int task = blockIdx.x * kGemvWarps + warp;
  if (task < n_tasks) {
    int r[ROWS];
    task_rows<ROWS>(EPI, task, p, r);
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const char* row = reinterpret_cast<const char*>(p.W + (size_t)r[i] * K);
      for (int off = lane * 128; off < K * 2; off += 32 * 128) prefetch_l2(row + off);
    }
  }
  grid_launch_dependents();
  grid_wait();
  DecodeState* st = p.st;
  if (st != nullptr && st->done) return;

  // ---- stage x (bf16) in shared memory ----
  if constexpr (IN == IN_X) {
    const uint4* src = reinterpret_cast<const uint4*>(p.x);
    for (int i = threadIdx.x; i < K / 8; i += kGemvThreads)
      reinterpret_cast<uint4*>(xs)[i] = src[i];
  } else {
    const float* hin = p.h;
    const __nv_bfloat16* erow = nullptr;
    if constexpr (IN == IN_EMBED_NORM) erow = p.embed + (size_t)st->token * K;
    float ss = 0.f;
    for (int i = threadIdx.x; i < K; i += kGemvThreads) {
      float v = (IN == IN_EMBED_NORM) ? bf_to_f(erow[i]) : hin[i];
      ss += v * v;
    }
    ss = block_sum(ss, red);
    const float rstd = rsqrtf(ss / K + p.eps);
    for (int i = threadIdx.x; i < K; i += kGemvThreads) {
      float v = (IN == IN_EMBED_NORM) ? bf_to_f(erow[i]) : hin[i];
      if constexpr (IN == IN_EMBED_NORM) {
        if (blockIdx.x == 0) p.h[i] = v;  // residual stream starts at the embedding
      }
      xs[i] = __float2bfloat16_rn(v * rstd * bf_to_f(p.norm_w[i]));
    }
  }
  __syncthreads();

  Top2 best;
  best.init();
  const uint4* xs4 = reinterpret_cast<const uint4*>(xs);

  for (; task < n_tasks; task += stride) {
    int r[ROWS];
    task_rows<ROWS>(EPI, task, p, r);
    float acc[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) acc[i] = 0.f;
    for (int c0 = 0; c0 < nchunk; c0 += U) {
      uint4 w[ROWS][U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = (c0 + u) * kChunk + lane * 8;
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
          w[i][u] = (c0 + u < nchunk && k < K) ? ld_stream(p.W + (size_t)r[i] * K + k)
                                               : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = (c0 + u) * kChunk + lane * 8;
        if (c0 + u < nchunk && k < K) {
          const uint4 xv = xs4[k / 8];
#pragma unroll
          for (int i = 0; i < ROWS; ++i) acc[i] = dot8(w[i][u], xv, acc[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < ROWS; ++i) acc[i] = warp_sum(acc[i]);

    if (lane == 0) {
      if constexpr (EPI == EPI_RESID) {
#pragma unroll
        for (int i = 0; i < ROWS; ++i) p.h[r[i]] += acc[i];
      } else if constexpr (EPI == EPI_LOGITS) {
#pragma unroll
        for (int i = 0; i < ROWS; ++i) p.logits[r[i]] = acc[i];
      } else if constexpr (EPI == EPI_ARGMAX) {
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
          if (r[i] < p.n_valid) best.push(acc[i], r[i]);
      } else if constexpr (EPI == EPI_GLU) {
        const float g = acc[0], u = acc[1];
        const float a = g / (1.f + __expf(-g)) * u;
        p.act_out[task] = __float2bfloat16_rn(a);
      } else if constexpr (EPI == EPI_QKV) {
        const int pos = st->pos;
        float v0 = acc[0] + bf_to_f(p.bias[r[0]]);
        float v1 = acc[1] + bf_to_f(p.bias[r[1]]);
        const int qk = p.q_dim + p.kv_dim;
        if (r[0] < qk) {
          const int j = r[0] % kHeadDim;  // < 64
          const float c = p.rope[((size_t)pos * kHalf + j) * 2];
          const float s = p.rope[((size_t)pos * kHalf + j) * 2 + 1];
          const float y0 = v0 * c - v1 * s;
          const float y1 = v1 * c + v0 * s;
          if (r[0] < p.q_dim) {
            p.qout[r[0]] = __float2bfloat16_rn(y0);
            p.qout[r[1]] = __float2bfloat16_rn(y1);
          } else {
            const int kvh = (r[0] - p.q_dim) / kHeadDim;
            const int page = st->page_table[pos / kPage];
            const size_t base = kv_offset(p.layer, page, kvh, pos % kPage, p.n_pages, p.n_kv);
            p.k_pool[base + j] = __float2bfloat16_rn(y0);
            p.k_pool[base + j + kHalf] = __float2bfloat16_rn(y1);
          }
        } else {
          const int vr = r[0] - qk;  // even
          const int kvh = vr / kHeadDim, dd = vr % kHeadDim;
          const int page = st->page_table[pos / kPage];
          const size_t base = kv_offset(p.layer, page, kvh, pos % kPage, p.n_pages, p.n_kv);
          p.v_pool[base + dd] = __float2bfloat16_rn(v0);
          p.v_pool[base + dd + 1] = __float2bfloat16_rn(v1);
        }
      }
    }
  }

  if constexpr (EPI == EPI_ARGMAX) {
    // CTA reduction -> partial; the last CTA selects the token
    if (lane == 0) { s_v1[warp] = best.v1; s_v2[warp] = best.v2; s_i1[warp] = best.i1; }
    __syncthreads();
    if (threadIdx.x == 0) {
      Top2 b;
      b.init();
      for (int w = 0; w < kGemvWarps; ++w) b.merge(s_v1[w], s_i1[w], s_v2[w]);
      p.part_v1[blockIdx.x] = b.v1;
      p.part_v2[blockIdx.x] = b.v2;
      p.part_i1[blockIdx.x] = b.i1;
      __threadfence();
      const unsigned prev = atomicAdd(p.counter, 1u);
      s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      Top2 b;
      b.init();
      for (int i = threadIdx.x; i < (int)gridDim.x; i += kGemvThreads) {
        b.merge(__ldcg(p.part_v1 + i), __ldcg(p.part_i1 + i), __ldcg(p.part_v2 + i));
      }
      warp_top2(b);
      if (lane == 0) { s_v1[warp] = b.v1; s_v2[warp] = b.v2; s_i1[warp] = b.i1; }
      __syncthreads();
      if (threadIdx.x == 0) {
        Top2 f;
        f.init();
        for (int w = 0; w < kGemvWarps; ++w) f.merge(s_v1[w], s_i1[w], s_v2[w]);
        *p.counter = 0u;
        select_token(st, f.i1, f.v1 - f.v2);
      }
    }
  }
}

// ------------------------------------------------------------- launchers ---
template <int IN, int EPI, int ROWS, int U>
static cudaError_t launch(const GemvParams& p, int grid, cudaStream_t stream, bool pdl) {
  const int smem = ((p.K * 2 + 15) / 16) * 16;
  auto fn = gemv_kernel<IN, EPI, ROWS, U>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kGemvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, p);
}

static int grid_for(int n_tasks, int num_sms, int per_sm) {
  int g = (n_tasks + kGemvWarps - 1) / kGemvWarps;
  const int cap = num_sms * per_sm;
  return g < cap ? g : cap;
}

cudaError_t gemv_launch(GemvKind kind, GemvParams p, int num_sms, cudaStream_t stream, bool pdl) {
  switch (kind) {
    case GEMV_QKV_EMBED:
      p.n_tasks = p.N / 2;
      return launch<IN_EMBED_NORM, EPI_QKV, 2, 4>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
    case GEMV_QKV:
      p.n_tasks = p.N / 2;
      return launch<IN_H_NORM, EPI_QKV, 2, 4>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
    case GEMV_RESID:
      p.n_tasks = p.N;
      return launch<IN_X, EPI_RESID, 1, 8>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
    case GEMV_GLU:
      p.n_tasks = p.N / 2;
      return launch<IN_H_NORM, EPI_GLU, 2, 4>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
    case GEMV_LM_ARGMAX:
      p.n_tasks = (p.n_valid + 1) / 2;
      return launch<IN_H_NORM, EPI_ARGMAX, 2, 4>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
    case GEMV_LM_ARGMAX_X:
      p.n_tasks = (p.n_valid + 1) / 2;
      return launch<IN_X, EPI_ARGMAX, 2, 4>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
    case GEMV_LM_LOGITS_X:
      p.n_tasks = (p.N + 1) / 2;
      return launch<IN_X, EPI_LOGITS, 2, 4>(p, grid_for(p.n_tasks, num_sms, 2), stream, pdl);
  }
  return cudaErrorInvalidValue;
}

int gemv_max_grid(int num_sms) { return num_sms * 2; }

}  // namespace sr
