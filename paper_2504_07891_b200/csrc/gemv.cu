// Decode-path GEMVs (batch-1 token): HBM-bound weight streaming with fused
// prologues (RMSNorm, embedding gather) and epilogues (bias + RoPE + K/V page
// append, residual add, SiLU*up, greedy argmax + stop test).
//
// Layout: W is row-major [N, K] bf16 (out_features x in_features).  A CTA of
// 8 warps stages the input vector x (bf16, K elements) in shared memory.  The
// CTA's warps form RG = 8 / KS row groups of KS warps; a row group owns a task
// of ROWS rows and its KS warps each stream one K-slice of those rows.
//
// Each warp walks a flat sequence of load batches (task, U chunks of 256
// elements) with two register buffers: batch b+1 is in flight while batch b is
// consumed, across task boundaries, so every warp keeps U*ROWS 16-byte
// ld.global.nc.L1::no_allocate loads outstanding for its whole lifetime.  The
// first batch depends only on the (constant) weights and is issued *before*
// the programmatic-dependent-launch wait, overlapping the previous kernel's
// tail.  fp32 accumulation, warp-shuffle reduction and, for KS > 1, a
// fixed-order shared-memory reduction of the K slices (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace sr {

enum { IN_X = 0, IN_H_NORM = 1, IN_EMBED_NORM = 2 };
enum { EPI_QKV = 0, EPI_RESID = 1, EPI_GLU = 2, EPI_ARGMAX = 3, EPI_LOGITS = 4 };

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;
constexpr int kChunk = 256;            // elements per warp-wide 16-byte load
constexpr int kNormMax = 5120 / kGemvThreads;  // h elements per thread (d <= 5120)
constexpr int kMaxIters = 32;          // K-split kernels: tasks per row group per CTA

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

template <int IN, int EPI, int ROWS, int U, int KS>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(GemvParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __shared__ float red[32];
  __shared__ float kpart[KS > 1 ? kMaxIters : 1][kGemvWarps / KS][KS];
  __shared__ float s_v1[kGemvWarps], s_v2[kGemvWarps];
  __shared__ int s_i1[kGemvWarps];
  __shared__ bool s_last;
  constexpr int RG = kGemvWarps / KS;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rg = warp / KS, ks = warp % KS;
  const int K = p.K;
  const int n_tasks = p.n_tasks;
  const int nchunk = (K + kChunk - 1) / kChunk;
  const int c_per = (nchunk + KS - 1) / KS;  // chunks of this warp's K slice
  const int c_lo = ks * c_per;
  const int c_hi = min(nchunk, c_lo + c_per);
  const int nb = c_hi > c_lo ? (c_hi - c_lo + U - 1) / U : 1;  // load batches per task
  const int stride = gridDim.x * RG;
  const int task0 = blockIdx.x * RG + rg;
  const int iters = (n_tasks + stride - 1) / stride;  // per CTA (uniform)
  const int my_iters = task0 < n_tasks ? (n_tasks - task0 + stride - 1) / stride : 0;
  const int total = my_iters * nb;

  uint4 wa[ROWS][U], wb[ROWS][U];
  auto load = [&](int B, uint4 (&w)[ROWS][U]) {
    const int task = task0 + (B / nb) * stride;
    const int c0 = c_lo + (B % nb) * U;
    int r[ROWS];
    task_rows<ROWS>(EPI, task, p, r);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = (c0 + u) * kChunk + lane * 8;
      const bool ok = (c0 + u < c_hi) && k < K;
#pragma unroll
      for (int i = 0; i < ROWS; ++i)
        w[i][u] = ok ? ld_stream(p.W + (size_t)r[i] * K + k) : make_uint4(0, 0, 0, 0);
    }
  };

  // ---- first weight batch: independent of every predecessor ----
  if (total > 0) load(0, wa);
  if (p.prefetch && total > 1) {
    int r[ROWS];
    task_rows<ROWS>(EPI, task0, p, r);
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const char* row = reinterpret_cast<const char*>(p.W + (size_t)r[i] * K);
      for (int c = c_lo + U + lane / 4; c < c_hi; c += 8)
        prefetch_l2(row + c * kChunk * 2 + (lane & 3) * 128);
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
    // RMSNorm of h (or of the embedding row): one read, values kept in registers
    float hv[kNormMax];
    const __nv_bfloat16* erow = nullptr;
    if constexpr (IN == IN_EMBED_NORM) erow = p.embed + (size_t)st->token * K;
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kNormMax; ++j) {
      const int i = threadIdx.x + j * kGemvThreads;
      float v = 0.f;
      if (i < K) v = (IN == IN_EMBED_NORM) ? bf_to_f(erow[i]) : p.h[i];
      hv[j] = v;
      ss += v * v;
    }
    ss = block_sum(ss, red);
    const float rstd = rsqrtf(ss / K + p.eps);
#pragma unroll
    for (int j = 0; j < kNormMax; ++j) {
      const int i = threadIdx.x + j * kGemvThreads;
      if (i < K) {
        if constexpr (IN == IN_EMBED_NORM) {
          if (blockIdx.x == 0) p.h[i] = hv[j];  // residual stream starts at the embedding
        }
        xs[i] = __float2bfloat16_rn(hv[j] * rstd * bf_to_f(p.norm_w[i]));
      }
    }
  }
  __syncthreads();

  Top2 best;
  best.init();
  const uint4* xs4 = reinterpret_cast<const uint4*>(xs);
  float acc[ROWS];
#pragma unroll
  for (int i = 0; i < ROWS; ++i) acc[i] = 0.f;

  auto finish = [&](int it) {
    const int task = task0 + it * stride;
#pragma unroll
    for (int i = 0; i < ROWS; ++i) acc[i] = warp_sum(acc[i]);
    if constexpr (KS > 1) {
      // park the K-slice partial; the CTA reduces all of them after the loop
      if (lane == 0 && it < kMaxIters) kpart[it][rg][ks] = acc[0];
    } else if (lane == 0) {
      int r[ROWS];
      task_rows<ROWS>(EPI, task, p, r);
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
        p.act_out[task] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * u);
      } else if constexpr (EPI == EPI_QKV) {
        const int pos = st->pos;
        const float v0 = acc[0] + bf_to_f(p.bias[r[0]]);
        const float v1 = acc[1] + bf_to_f(p.bias[r[1]]);
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
#pragma unroll
    for (int i = 0; i < ROWS; ++i) acc[i] = 0.f;
  };

  auto consume = [&](int B, const uint4 (&w)[ROWS][U]) {
    const int cb = B % nb;
    const int c0 = c_lo + cb * U;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = (c0 + u) * kChunk + lane * 8;
      if (c0 + u < c_hi && k < K) {
        const uint4 xv = xs4[k / 8];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) acc[i] = dot8(w[i][u], xv, acc[i]);
      }
    }
    if (cb == nb - 1) finish(B / nb);
  };

  // ---- software-pipelined stream: two register buffers ----
  for (int B = 0; B < total; B += 2) {
    if (B + 1 < total) load(B + 1, wb);
    consume(B, wa);
    if (B + 1 < total) {
      if (B + 2 < total) load(B + 2, wa);
      consume(B + 1, wb);
    }
  }

  if constexpr (KS > 1) {
    // fixed-order reduction of the K-slice partials, then the residual epilogue
    static_assert(EPI == EPI_RESID && ROWS == 1, "K-split is for residual GEMVs");
    __syncthreads();
    const int n_out = min(iters, kMaxIters) * RG;
    for (int o = threadIdx.x; o < n_out; o += kGemvThreads) {
      const int oit = o / RG, org = o % RG;
      const int task = blockIdx.x * RG + org + oit * stride;
      if (task >= n_tasks) continue;
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < KS; ++j) s += kpart[oit][org][j];
      p.h[task] += s;
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
      for (int i = threadIdx.x; i < (int)gridDim.x; i += kGemvThreads)
        b.merge(__ldcg(p.part_v1 + i), __ldcg(p.part_i1 + i), __ldcg(p.part_v2 + i));
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
template <int IN, int EPI, int ROWS, int U, int KS>
static cudaError_t launch(const GemvParams& p, int grid, cudaStream_t stream, bool pdl) {
  const int smem = ((p.K * 2 + 15) / 16) * 16;
  auto fn = gemv_kernel<IN, EPI, ROWS, U, KS>;
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

static int gemv_per_sm() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SR_GEMV_PER_SM");
    v = e ? atoi(e) : 4;
    if (v < 1 || v > 4) v = 4;
  }
  return v;
}

static int grid_for(int n_tasks, int rows_per_cta, int num_sms) {
  int g = (n_tasks + rows_per_cta - 1) / rows_per_cta;
  const int cap = num_sms * gemv_per_sm();
  return g < cap ? g : cap;
}

// chunks per load batch: SR_GEMV_U (pair kernels) / SR_GEMV_UR (residual) tune
static int env_u(const char* name, int dflt) {
  const char* e = getenv(name);
  const int v = e ? atoi(e) : dflt;
  return (v == 2 || v == 4 || v == 8) ? v : dflt;
}

template <int IN, int EPI, int ROWS, int U>
static cudaError_t launch1(GemvParams p, int num_sms, cudaStream_t stream, bool pdl) {
  static const int u = env_u("SR_GEMV_U", U);
  const int grid = grid_for(p.n_tasks, kGemvWarps, num_sms);
  if (u == 8) return launch<IN, EPI, ROWS, 8, 1>(p, grid, stream, pdl);
  if (u == 2) return launch<IN, EPI, ROWS, 2, 1>(p, grid, stream, pdl);
  return launch<IN, EPI, ROWS, 4, 1>(p, grid, stream, pdl);
}

template <int U>
static cudaError_t launch_resid_u(GemvParams p, int ks, int num_sms, cudaStream_t stream, bool pdl) {
  switch (ks) {
    case 1: return launch<IN_X, EPI_RESID, 1, U, 1>(p, grid_for(p.n_tasks, kGemvWarps, num_sms), stream, pdl);
    case 2: return launch<IN_X, EPI_RESID, 1, U, 2>(p, grid_for(p.n_tasks, kGemvWarps / 2, num_sms), stream, pdl);
    case 4: return launch<IN_X, EPI_RESID, 1, U, 4>(p, grid_for(p.n_tasks, kGemvWarps / 4, num_sms), stream, pdl);
    default: return launch<IN_X, EPI_RESID, 1, U, 8>(p, grid_for(p.n_tasks, 1, num_sms), stream, pdl);
  }
}

static cudaError_t launch_resid(GemvParams p, int ks, int num_sms, cudaStream_t stream, bool pdl) {
  static const int u = env_u("SR_GEMV_UR", 4);
  if (u == 8) return launch_resid_u<8>(p, ks, num_sms, stream, pdl);
  if (u == 2) return launch_resid_u<2>(p, ks, num_sms, stream, pdl);
  return launch_resid_u<4>(p, ks, num_sms, stream, pdl);
}

// K-split for one-row-per-task residual GEMVs: split while the chip has fewer
// than ~4 row tasks per warp slot and each slice keeps >= 4 chunks per warp
static int pick_ks(int rows, int K, int num_sms) {
  const int slots = num_sms * gemv_per_sm() * kGemvWarps;
  const int nchunk = K / kChunk;
  int ks = 1;
  while (ks < 8 && (long)rows * ks < 4L * slots && nchunk / (ks * 2) >= 4) ks *= 2;
  return ks;
}

cudaError_t gemv_launch(GemvKind kind, GemvParams p, int num_sms, cudaStream_t stream, bool pdl) {
  if (p.K > 5120 && (kind == GEMV_QKV || kind == GEMV_QKV_EMBED || kind == GEMV_GLU ||
                     kind == GEMV_LM_ARGMAX || kind == GEMV_LM_LOGITS))
    return cudaErrorInvalidValue;  // RMSNorm prologue keeps d <= 5120 values in registers
  switch (kind) {
    case GEMV_QKV_EMBED:
      p.n_tasks = p.N / 2;
      return launch1<IN_EMBED_NORM, EPI_QKV, 2, 4>(p, num_sms, stream, pdl);
    case GEMV_QKV:
      p.n_tasks = p.N / 2;
      return launch1<IN_H_NORM, EPI_QKV, 2, 4>(p, num_sms, stream, pdl);
    case GEMV_RESID: {
      p.n_tasks = p.N;
      int ks = pick_ks(p.N, p.K, num_sms);
      const int rg = kGemvWarps / ks;
      const int grid = grid_for(p.N, rg, num_sms);
      if ((p.N + grid * rg - 1) / (grid * rg) > kMaxIters) ks = 1;  // partial buffer bound
      return launch_resid(p, ks, num_sms, stream, pdl);
    }
    case GEMV_GLU:
      p.n_tasks = p.N / 2;
      return launch1<IN_H_NORM, EPI_GLU, 2, 4>(p, num_sms, stream, pdl);
    case GEMV_LM_ARGMAX:
      p.n_tasks = (p.n_valid + 1) / 2;
      return launch1<IN_H_NORM, EPI_ARGMAX, 2, 4>(p, num_sms, stream, pdl);
    case GEMV_LM_ARGMAX_X:
      p.n_tasks = (p.n_valid + 1) / 2;
      return launch1<IN_X, EPI_ARGMAX, 2, 4>(p, num_sms, stream, pdl);
    case GEMV_LM_LOGITS_X:
      p.n_tasks = (p.N + 1) / 2;
      return launch1<IN_X, EPI_LOGITS, 2, 4>(p, num_sms, stream, pdl);
    case GEMV_LM_LOGITS:
      p.n_tasks = (p.N + 1) / 2;
      return launch1<IN_H_NORM, EPI_LOGITS, 2, 4>(p, num_sms, stream, pdl);
  }
  return cudaErrorInvalidValue;
}

int gemv_max_grid(int num_sms) { return num_sms * 4; }

}  // namespace sr
