// Prefill path (prompt suffixes and verification passes, M >= 1 tokens):
// embedding + RMSNorm, split-K GEMM partials, and the reduce-epilogues that
// finish each projection (bias + RoPE + K/V page append; residual add fused
// with the next RMSNorm; SiLU * up), plus the verify readout (K8).
#include "common.cuh"
#include "kernels.h"

namespace sr {

// ========================================================= epilogues ======
constexpr int kEpiThreads = 256;
constexpr int kEpiRowThreads = 1024;  // one CTA per token row: wide, for latency

// launch with programmatic dependent launch: the kernel starts while its
// predecessor drains and calls grid_wait() before touching its outputs
template <typename... Args, typename... Actual>
static cudaError_t launch_pdl(void (*fn)(Args...), dim3 grid, int block, size_t smem,
                              cudaStream_t stream, Actual... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, args...);
}

// h[m] = embed[ids[m]];  x[m] = bf16(rmsnorm(h[m]) * w)
__global__ void embed_norm_kernel(const int* ids, const __nv_bfloat16* embed, int d,
                                  const __nv_bfloat16* w, float eps, float* h, __nv_bfloat16* x) {
  __shared__ float red[32];
  const int m = blockIdx.x;
  const __nv_bfloat16* e = embed + (size_t)ids[m] * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = bf_to_f(e[i]);
    h[(size_t)m * d + i] = v;
    ss += v * v;
  }
  ss = block_sum(ss, red);
  const float rstd = rsqrtf(ss / d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    x[(size_t)m * d + i] = __float2bfloat16_rn(bf_to_f(e[i]) * rstd * bf_to_f(w[i]));
}

cudaError_t embed_norm_launch(const int* ids, int M, const __nv_bfloat16* embed, int d,
                              const __nv_bfloat16* norm_w, float eps, float* h,
                              __nv_bfloat16* x, cudaStream_t stream) {
  embed_norm_kernel<<<M, kEpiThreads, 0, stream>>>(ids, embed, d, norm_w, eps, h, x);
  return cudaGetLastError();
}

// fixed-order sum of the split-K partials; the (<= 8) loads are independent
// predicated loads, so they are all in flight together
SR_DEV float sum_splits(const float* part, int splits, size_t stride, size_t idx) {
  float a[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) a[s] = s < splits ? __ldcg(part + s * stride + idx) : 0.f;
  float v = 0.f;
#pragma unroll
  for (int s = 0; s < 8; ++s) v += a[s];
  return v;
}

// 4 consecutive outputs: sum over the splits (same order as sum_splits) + bias
SR_DEV float4 sum_splits4_bias(const float* part, int splits, size_t stride, size_t idx,
                               const __nv_bfloat16* bias) {
  float4 a[8];
#pragma unroll
  for (int sp = 0; sp < 8; ++sp)
    a[sp] = sp < splits ? __ldcg(reinterpret_cast<const float4*>(part + sp * stride + idx))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int sp = 0; sp < 8; ++sp) {
    t.x += a[sp].x;
    t.y += a[sp].y;
    t.z += a[sp].z;
    t.w += a[sp].w;
  }
  const uint2 b = *reinterpret_cast<const uint2*>(bias);
  const float2 b01 = bf2_to_f2(b.x), b23 = bf2_to_f2(b.y);
  return make_float4(t.x + b01.x, t.y + b01.y, t.z + b23.x, t.w + b23.y);
}

SR_DEV void store_bf16x4(__nv_bfloat16* dst, float a, float b, float c, float d) {
  *reinterpret_cast<uint2*>(dst) = make_uint2(f2_to_bf2(a, b), f2_to_bf2(c, d));
}

// q/k: bias + RoPE (pairs j, j+64); k, v -> pages; q -> bf16 buffer.
// A thread takes 4 rotation pairs (or 4 v values): 16-byte partial loads.
__global__ void epi_qkv_kernel(EpiParams p) {
  grid_launch_dependents();
  grid_wait();
  const int m = blockIdx.x;
  const int pos = p.tok_meta ? p.tok_meta[2 * m] : p.start_pos + m;
  const size_t stride = (size_t)p.M * p.N;
  const int qk = p.q_dim + p.kv_dim;
  const int nq4 = qk / 8, nv4 = p.kv_dim / 4;
  const int page = p.tok_meta ? p.tok_meta[2 * m + 1] : p.page_table[pos / kPage];
  const size_t row = (size_t)m * p.N;
  for (int t = blockIdx.y * blockDim.x + threadIdx.x; t < nq4 + nv4; t += gridDim.y * blockDim.x) {
    if (t < nq4) {
      const int j = (t % (kHalf / 4)) * 4;
      const int r0 = (t / (kHalf / 4)) * kHeadDim + j, r1 = r0 + kHalf;
      const float4 v0 = sum_splits4_bias(p.part, p.splits, stride, row + r0, p.bias + r0);
      const float4 v1 = sum_splits4_bias(p.part, p.splits, stride, row + r1, p.bias + r1);
      const float4* rp = reinterpret_cast<const float4*>(p.rope + ((size_t)pos * kHalf + j) * 2);
      const float4 cs01 = rp[0], cs23 = rp[1];  // (c, s) of j .. j+3
      const float y0[4] = {v0.x * cs01.x - v1.x * cs01.y, v0.y * cs01.z - v1.y * cs01.w,
                           v0.z * cs23.x - v1.z * cs23.y, v0.w * cs23.z - v1.w * cs23.w};
      const float y1[4] = {v1.x * cs01.x + v0.x * cs01.y, v1.y * cs01.z + v0.y * cs01.w,
                           v1.z * cs23.x + v0.z * cs23.y, v1.w * cs23.z + v0.w * cs23.w};
      __nv_bfloat16 *d0, *d1;
      if (r0 < p.q_dim) {
        d0 = p.q + (size_t)m * p.q_dim + r0;
        d1 = d0 + kHalf;
      } else {
        const int kvh = (r0 - p.q_dim) / kHeadDim;
        d0 = p.k_pool + kv_offset(p.layer, page, kvh, pos % kPage, p.n_pages, p.n_kv) + j;
        d1 = d0 + kHalf;
      }
      store_bf16x4(d0, y0[0], y0[1], y0[2], y0[3]);
      store_bf16x4(d1, y1[0], y1[1], y1[2], y1[3]);
    } else {
      const int vr = 4 * (t - nq4), kvh = vr / kHeadDim, dd = vr % kHeadDim;
      const float4 v = sum_splits4_bias(p.part, p.splits, stride, row + qk + vr, p.bias + qk + vr);
      store_bf16x4(p.v_pool + kv_offset(p.layer, page, kvh, pos % kPage, p.n_pages, p.n_kv) + dd,
                   v.x, v.y, v.z, v.w);
    }
  }
}

cudaError_t epi_qkv_launch(const EpiParams& p, cudaStream_t stream) {
  // a row's (4-pair / 4-value) groups spread over 256-thread CTAs: short verify
  // passes still put several CTAs per row in flight
  const int groups = (p.q_dim + p.kv_dim) / 8 + p.kv_dim / 4;
  return launch_pdl(epi_qkv_kernel, dim3(p.M, (groups + 255) / 256), 256, 0, stream, p);
}

// h[m] += sum_s part;  x[m] = bf16(rmsnorm(h[m]) * w)   (N == d, d % 4 == 0)
// 16-byte loads of h and of every split's partial; same summation order as
// sum_splits (splits 0..7 in turn, then added to h)
__global__ void epi_resid_norm_kernel(EpiParams p) {
  grid_launch_dependents();
  grid_wait();
  extern __shared__ float hrow[];
  __shared__ float red[32];
  const int m = blockIdx.x, d = p.N;
  const size_t stride = (size_t)p.M * p.N;
  float4* h4 = reinterpret_cast<float4*>(p.h + (size_t)m * d);
  float ss = 0.f;
  for (int i = threadIdx.x; i < (d >> 2); i += blockDim.x) {
    const size_t idx = (size_t)m * d + 4 * (size_t)i;
    float4 a[8];
#pragma unroll
    for (int sp = 0; sp < 8; ++sp)
      a[sp] = sp < p.splits ? __ldcg(reinterpret_cast<const float4*>(p.part + sp * stride + idx))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int sp = 0; sp < 8; ++sp) {
      t.x += a[sp].x;
      t.y += a[sp].y;
      t.z += a[sp].z;
      t.w += a[sp].w;
    }
    float4 v = h4[i];
    v.x += t.x;
    v.y += t.y;
    v.z += t.z;
    v.w += t.w;
    h4[i] = v;
    reinterpret_cast<float4*>(hrow)[i] = v;
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = block_sum(ss, red);
  const float rstd = rsqrtf(ss / d + p.eps);
  const uint2* w4 = reinterpret_cast<const uint2*>(p.norm_w);
  uint2* x4 = reinterpret_cast<uint2*>(p.x + (size_t)m * d);
  for (int i = threadIdx.x; i < (d >> 2); i += blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(hrow)[i];
    const uint2 w = w4[i];
    const float2 w01 = bf2_to_f2(w.x), w23 = bf2_to_f2(w.y);
    x4[i] = make_uint2(f2_to_bf2(v.x * rstd * w01.x, v.y * rstd * w01.y),
                       f2_to_bf2(v.z * rstd * w23.x, v.w * rstd * w23.y));
  }
}

cudaError_t epi_resid_norm_launch(const EpiParams& p, cudaStream_t stream) {
  // few rows: wide CTAs keep many loads in flight per row; many rows (batched
  // verify): 256 threads, so that every row is resident in one wave
  const int threads = p.M >= 256 ? 256 : kEpiRowThreads;
  return launch_pdl(epi_resid_norm_kernel, dim3(p.M), threads, p.N * sizeof(float), stream, p);
}

// act[m][u] = bf16(silu(gate) * up) from interleaved 16-row blocks
__global__ void epi_glu_kernel(EpiParams p) {
  grid_launch_dependents();
  grid_wait();
  const int m = blockIdx.y;
  const int f = p.N / 2;
  const size_t stride = (size_t)p.M * p.N;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < f; u += gridDim.x * blockDim.x) {
    const int b = u >> 4, j = u & 15;
    const float g = sum_splits(p.part, p.splits, stride, (size_t)m * p.N + 32 * b + j);
    const float v = sum_splits(p.part, p.splits, stride, (size_t)m * p.N + 32 * b + 16 + j);
    p.act[(size_t)m * f + u] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * v);
  }
}

cudaError_t epi_glu_launch(const EpiParams& p, cudaStream_t stream) {
  const int f = p.N / 2;
  dim3 grid((f + kEpiThreads - 1) / kEpiThreads, p.M);
  return launch_pdl(epi_glu_kernel, grid, kEpiThreads, 0, stream, p);
}

// ================================================ per-row greedy choices ====
// rows x vocab logits (sum of split partials) -> argmax (ties: lower id) and
// top-1 minus top-2 margin per row; one CTA per row
__global__ void __launch_bounds__(1024) rows_argmax_kernel(const float* part, int splits,
                                                           size_t stride, int N, int n_valid,
                                                           int base, int32_t* out_ids,
                                                           float* margins) {
  grid_wait();
  __shared__ float s1[32], s2[32];
  __shared__ int si[32];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Top2 b;
  b.init();
  for (int v = tid; v < n_valid; v += blockDim.x) {
    float x = 0.f;
    for (int sp = 0; sp < splits; ++sp) x += __ldcg(part + sp * stride + (size_t)r * N + v);
    b.push(x, base + v);
  }
  warp_top2(b);
  if (lane == 0) { s1[warp] = b.v1; s2[warp] = b.v2; si[warp] = b.i1; }
  __syncthreads();
  if (tid == 0) {
    Top2 f;
    f.init();
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) f.merge(s1[w], si[w], s2[w]);
    out_ids[r] = f.i1;
    if (margins) margins[r] = f.v1 - f.v2;
  }
}

// Few rows (batched decode steps): each row's vocabulary is split over
// kArgmaxChunks CTAs; the last CTA of a row merges the chunk top-2s in chunk
// order (deterministic, ties: lower id) and resets the row's counter.
constexpr int kArgmaxChunks = 16;
__global__ void __launch_bounds__(512) rows_argmax_chunk_kernel(
    const float* part, int splits, size_t stride, int N, int n_valid, int base, int32_t* out_ids,
    float* margins, float* cv1, float* cv2, int* ci1, unsigned* ctr) {
  grid_wait();
  __shared__ float s1[16], s2[16];
  __shared__ int si[16];
  __shared__ bool last;
  const int r = blockIdx.x, c = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n_valid + kArgmaxChunks - 1) / kArgmaxChunks;
  const int v0 = c * per, v1 = min(n_valid, v0 + per);
  Top2 b;
  b.init();
  for (int v = v0 + tid; v < v1; v += blockDim.x) {
    float x = 0.f;
    for (int sp = 0; sp < splits; ++sp) x += __ldcg(part + sp * stride + (size_t)r * N + v);
    b.push(x, base + v);
  }
  warp_top2(b);
  if (lane == 0) { s1[warp] = b.v1; s2[warp] = b.v2; si[warp] = b.i1; }
  __syncthreads();
  if (tid == 0) {
    Top2 f;
    f.init();
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) f.merge(s1[w], si[w], s2[w]);
    const int k = r * kArgmaxChunks + c;
    cv1[k] = f.v1;
    cv2[k] = f.v2;
    ci1[k] = f.i1;
    __threadfence();
    last = atomicAdd(ctr + r, 1u) == kArgmaxChunks - 1;
  }
  __syncthreads();
  if (!last || tid != 0) return;
  __threadfence();
  Top2 f;
  f.init();
  for (int k = r * kArgmaxChunks; k < (r + 1) * kArgmaxChunks; ++k)
    f.merge(__ldcg(cv1 + k), __ldcg(ci1 + k), __ldcg(cv2 + k));
  out_ids[r] = f.i1;
  if (margins) margins[r] = f.v1 - f.v2;
  ctr[r] = 0u;
}

cudaError_t rows_argmax_launch(const float* part, int splits, size_t stride, int rows, int N,
                               int n_valid, int base, int32_t* out_ids, float* margins,
                               cudaStream_t stream, float* cv1, float* cv2, int* ci1,
                               unsigned* ctr, int scratch) {
  if (cv1 && rows * kArgmaxChunks <= scratch && rows <= 16)
    return launch_pdl(rows_argmax_chunk_kernel, dim3(rows, kArgmaxChunks), 512, 0, stream, part,
                      splits, stride, N, n_valid, base, out_ids, margins, cv1, cv2, ci1, ctr);
  return launch_pdl(rows_argmax_kernel, dim3(rows), 1024, 0, stream, part, splits, stride, N,
                    n_valid, base, out_ids, margins);
}

// ======================================================= verify readout ====
// Pass 1 (grid-wide): greedy top-2 partials and, for each digit d, the count
// of valid ids ranked before it (logit greater, or equal with a lower id).
// The last CTA applies extract_score's preference order and the threshold.
constexpr int kReadoutThreads = 256;

__global__ void __launch_bounds__(kReadoutThreads) readout_kernel(ReadoutParams p) {
  __shared__ float dig[10];
  __shared__ unsigned int cnt[10];
  __shared__ float s_v1[8], s_v2[8];
  __shared__ int s_i1[8];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 10) { dig[tid] = p.logits[tid]; cnt[tid] = 0; }
  __syncthreads();
  float dl[10];
#pragma unroll
  for (int d = 0; d < 10; ++d) dl[d] = dig[d];
  unsigned int c[10];
#pragma unroll
  for (int d = 0; d < 10; ++d) c[d] = 0;
  Top2 best;
  best.init();
  for (int v = blockIdx.x * blockDim.x + tid; v < p.n_valid; v += gridDim.x * blockDim.x) {
    const float x = p.logits[v];
    best.push(x, v);
#pragma unroll
    for (int d = 0; d < 10; ++d) c[d] += (x > dl[d] || (x == dl[d] && v < d)) ? 1u : 0u;
  }
#pragma unroll
  for (int d = 0; d < 10; ++d) {
    unsigned int s = c[d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) atomicAdd(&cnt[d], s);
  }
  warp_top2(best);
  if (lane == 0) { s_v1[warp] = best.v1; s_v2[warp] = best.v2; s_i1[warp] = best.i1; }
  __syncthreads();
  if (tid == 0) {
    Top2 b;
    b.init();
    for (int w = 0; w < kReadoutThreads / 32; ++w) b.merge(s_v1[w], s_i1[w], s_v2[w]);
    p.part_v1[blockIdx.x] = b.v1;
    p.part_v2[blockIdx.x] = b.v2;
    p.part_i1[blockIdx.x] = b.i1;
    for (int d = 0; d < 10; ++d) atomicAdd(&p.counts[d], cnt[d]);
    __threadfence();
    const unsigned prev = atomicAdd(&p.counts[10], 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  __threadfence();
  Top2 g;
  g.init();
  for (int i = 0; i < (int)gridDim.x; ++i)
    g.merge(__ldcg(p.part_v1 + i), __ldcg(p.part_i1 + i), __ldcg(p.part_v2 + i));
  int best_d = -1;
  float best_v = -INFINITY, second = -INFINITY;
  for (int d = 0; d < 10; ++d) {
    const unsigned rank = __ldcg(&p.counts[d]);
    if (rank >= 10 || d >= p.n_valid) continue;
    const float v = dig[d];
    if (best_d < 0 || v > best_v) { second = best_v; best_v = v; best_d = d; }
    else if (v > second) second = v;
  }
  int score = best_d;
  if (score < 0) score = p.first_digit[g.i1];
  sr_readout r;
  r.score = score;
  r.accept = (score >= 0 && score >= p.threshold) ? 1 : 0;
  r.margin = best_d >= 0 ? best_v - second : 0.f;
  r.argmax = g.i1;
  *p.out = r;
  for (int d = 0; d <= 10; ++d) p.counts[d] = 0;
}

cudaError_t readout_launch(const ReadoutParams& p, int num_sms, cudaStream_t stream) {
  readout_kernel<<<num_sms, kReadoutThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

// ===================================================== decode bookkeeping ===
__global__ void decode_begin_kernel(DecodeState* st, DecodeState init, const int32_t* feed) {
  if (feed) init.token = feed[0];  // one fed token: the decode kernel processes it itself
  *st = init;
}

cudaError_t decode_begin_launch(DecodeState* st, const DecodeState* h_init, cudaStream_t stream,
                                const int32_t* feed) {
  decode_begin_kernel<<<1, 1, 0, stream>>>(st, *h_init, feed);
  return cudaGetLastError();
}

// First node of the decode graph: arm the while-loop from the prefill's choice.
__global__ void cond_init_kernel(DecodeState* st, unsigned long long handle) {
  st->cond_handle = handle;
  cudaGraphSetConditional((cudaGraphConditionalHandle)handle, st->done ? 0u : 1u);
}

cudaError_t cond_init_launch(DecodeState* st, unsigned long long handle, cudaStream_t stream) {
  cond_init_kernel<<<1, 1, 0, stream>>>(st, handle);
  return cudaGetLastError();
}

}  // namespace sr
