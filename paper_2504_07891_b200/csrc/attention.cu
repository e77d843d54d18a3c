// Paged GQA attention over the K/V page pools (flash-decoding split-KV).
//
// One CTA = (kv head g, KV split s, query row m).  Its 4 warps are split into
// 8 half-warp "streams"; a stream walks key positions lo+stream, lo+stream+8,
// ... of the split, each of its 16 lanes owning 8 of the 128 head dims (one
// 16-byte K load and one 16-byte V load per position, coalesced 256 B per
// half-warp).  All G = H/KV query heads of the group are processed together so
// each K/V byte is read once per query row.  Scores use exp2 with the log2(e)
// / sqrt(128) scale folded in; online softmax state (m, l, acc) is merged
// across streams in shared memory, written as a split partial, and the last
// CTA of (g, m) -- found with an atomic ticket -- merges the splits and writes
// the bf16 output.  Causality: query row m (absolute position start_pos + m)
// sees positions <= start_pos + m.
#include "common.cuh"
#include "kernels.h"

namespace sr {

constexpr int kAttnThreads = 128;
constexpr int kStreams = kAttnThreads / 16;
constexpr int kMaxGroup = 8;
constexpr int kMaxSplit = 64;    // grid.y <= kMaxSplit
constexpr int kMinChunk = 64;    // positions per split at least (one page)

template <int G>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(AttnParams p) {
  __shared__ float s_m[kStreams][G], s_l[kStreams][G];
  __shared__ float s_acc[kStreams][G][kHeadDim];
  __shared__ bool s_last;

  const bool decode = (p.st != nullptr);
  grid_launch_dependents();
  grid_wait();
  if (decode && p.st->done) return;

  const int g = blockIdx.x, split = blockIdx.y, m = blockIdx.z;
  const int tid = threadIdx.x, stream = tid >> 4, sl = tid & 15;
  const int T = decode ? p.st->ctx_len : p.start_pos + m + 1;
  const int* ptab = decode ? p.st->page_table : p.page_table;
  const int nsplit = p.nsplit;
  int chunk = (T + nsplit - 1) / nsplit;
  chunk = chunk < kMinChunk ? kMinChunk : ((chunk + 15) & ~15);
  const int lo = split * chunk;
  const int hi = min(T, lo + chunk);

  const int qdim = p.n_heads * kHeadDim;
  const float scale = 1.4426950408889634f * rsqrtf((float)kHeadDim);

  float q[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    const uint4 qv = *reinterpret_cast<const uint4*>(p.q + (size_t)m * qdim +
                                                       (size_t)(g * G + j) * kHeadDim + sl * 8);
    float2 a = bf2_to_f2(qv.x), b = bf2_to_f2(qv.y), c = bf2_to_f2(qv.z), d = bf2_to_f2(qv.w);
    q[j][0] = a.x * scale; q[j][1] = a.y * scale; q[j][2] = b.x * scale; q[j][3] = b.y * scale;
    q[j][4] = c.x * scale; q[j][5] = c.y * scale; q[j][6] = d.x * scale; q[j][7] = d.y * scale;
  }

  float mx[G], l[G], acc[G][8];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    mx[j] = -INFINITY;
    l[j] = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;
  }

  // The loop bound is warp-uniform (both half-warps iterate together) so the
  // full-mask shuffles below always see all 32 lanes; a half-warp whose
  // position is past `hi` computes on zeros and skips the state update.
  const int warp_first = lo + (stream & ~1);
  for (int i = 0; warp_first + i < hi; i += kStreams) {
    const int t = lo + stream + i;
    const bool valid = t < hi;
    uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
    if (valid) {
      const int page = ptab[t / kPage];
      const size_t off = kv_offset(p.layer, page, g, t % kPage, p.n_pages, p.n_kv) + sl * 8;
      kv = *reinterpret_cast<const uint4*>(p.k_pool + off);
      vv = *reinterpret_cast<const uint4*>(p.v_pool + off);
    }
    float k8[8], v8[8];
    {
      float2 a = bf2_to_f2(kv.x), b = bf2_to_f2(kv.y), c = bf2_to_f2(kv.z), d = bf2_to_f2(kv.w);
      k8[0] = a.x; k8[1] = a.y; k8[2] = b.x; k8[3] = b.y; k8[4] = c.x; k8[5] = c.y; k8[6] = d.x; k8[7] = d.y;
      a = bf2_to_f2(vv.x); b = bf2_to_f2(vv.y); c = bf2_to_f2(vv.z); d = bf2_to_f2(vv.w);
      v8[0] = a.x; v8[1] = a.y; v8[2] = b.x; v8[3] = b.y; v8[4] = c.x; v8[5] = c.y; v8[6] = d.x; v8[7] = d.y;
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fmaf(q[j][e], k8[e], s);
      s += __shfl_xor_sync(0xffffffffu, s, 8);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      if (!valid) continue;
      const float mn = fmaxf(mx[j], s);
      const float corr = exp2f(mx[j] - mn);
      const float pr = exp2f(s - mn);
      l[j] = l[j] * corr + pr;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] = fmaf(acc[j][e], corr, pr * v8[e]);
      mx[j] = mn;
    }
  }

  // ---- merge the 8 streams of this CTA ----
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (sl == 0) { s_m[stream][j] = mx[j]; s_l[stream][j] = l[j]; }
#pragma unroll
    for (int e = 0; e < 8; ++e) s_acc[stream][j][sl * 8 + e] = acc[j][e];
  }
  __syncthreads();

  const int n_rows = gridDim.z;
  const size_t part_stride = kHeadDim + 2;
  for (int idx = tid; idx < G * kHeadDim; idx += kAttnThreads) {
    const int j = idx / kHeadDim, d = idx % kHeadDim;
    float M = -INFINITY;
    for (int s = 0; s < kStreams; ++s) M = fmaxf(M, s_m[s][j]);
    float L = 0.f, A = 0.f;
    if (M != -INFINITY) {
      for (int s = 0; s < kStreams; ++s) {
        const float w = exp2f(s_m[s][j] - M);
        L += s_l[s][j] * w;
        A += s_acc[s][j][d] * w;
      }
    }
    float* part = p.part + (((size_t)m * p.n_heads + g * G + j) * nsplit + split) * part_stride;
    part[d] = A;
    if (d == 0) { part[kHeadDim] = M; part[kHeadDim + 1] = L; }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned int* ctr = p.counters + (size_t)m * p.n_kv + g;
    const unsigned prev = atomicAdd(ctr, 1u);
    s_last = (prev == (unsigned)nsplit - 1);
    if (s_last) *ctr = 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- last CTA of (g, m): merge the splits (parallel over splits) ----
  // 1) split weights w_s = exp2(m_s - M) / L into shared memory
  float* wsm = &s_acc[0][0][0];         // reuse: G * kMaxSplit split maxima -> weights
  float* lsm = wsm + G * kMaxSplit;     //        G * kMaxSplit split sums
  for (int idx = tid; idx < G * nsplit; idx += kAttnThreads) {
    const int j = idx / nsplit, sp = idx % nsplit;
    const float* ps = p.part + (((size_t)m * p.n_heads + g * G + j) * nsplit + sp) * part_stride;
    wsm[j * kMaxSplit + sp] = __ldcg(ps + kHeadDim);
    lsm[j * kMaxSplit + sp] = __ldcg(ps + kHeadDim + 1);
  }
  __syncthreads();
  if (tid < G) {
    const int j = tid;
    float M = -INFINITY;
    for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, wsm[j * kMaxSplit + sp]);
    float L = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float ms = wsm[j * kMaxSplit + sp];
      const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
      L += w * lsm[j * kMaxSplit + sp];
      wsm[j * kMaxSplit + sp] = w;
    }
    const float inv = 1.f / L;
    for (int sp = 0; sp < nsplit; ++sp) wsm[j * kMaxSplit + sp] *= inv;
  }
  __syncthreads();
  // 2) out[j][d] = sum_s w_s * acc_s[d]; independent loads, unrolled
  for (int idx = tid; idx < G * kHeadDim; idx += kAttnThreads) {
    const int j = idx / kHeadDim, d = idx % kHeadDim;
    const float* base = p.part + (((size_t)m * p.n_heads + g * G + j) * nsplit) * part_stride + d;
    float A = 0.f;
#pragma unroll 8
    for (int sp = 0; sp < nsplit; ++sp) {
      const float w = wsm[j * kMaxSplit + sp];
      if (w != 0.f) A = fmaf(w, __ldcg(base + sp * part_stride), A);
    }
    p.out[(size_t)m * qdim + (size_t)(g * G + j) * kHeadDim + d] = __float2bfloat16_rn(A);
  }
  (void)n_rows;
}

template <int G>
static cudaError_t launch_g(const AttnParams& p, int M, cudaStream_t stream, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_kv, p.nsplit, M);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_kernel<G>, p);
}

static cudaError_t launch_any(const AttnParams& p, int M, cudaStream_t stream, bool pdl) {
  switch (p.n_heads / p.n_kv) {
    case 1: return launch_g<1>(p, M, stream, pdl);
    case 2: return launch_g<2>(p, M, stream, pdl);
    case 4: return launch_g<4>(p, M, stream, pdl);
    case 5: return launch_g<5>(p, M, stream, pdl);
    case 6: return launch_g<6>(p, M, stream, pdl);
    case 7: return launch_g<7>(p, M, stream, pdl);
    case 8: return launch_g<8>(p, M, stream, pdl);
  }
  return cudaErrorInvalidValue;
}

int attn_decode_splits(int n_kv, int num_sms) {
  int s = (num_sms + n_kv - 1) / n_kv;  // ~one CTA per SM at long contexts
  return s < 1 ? 1 : (s > kMaxSplit ? kMaxSplit : s);
}

int attn_prefill_splits(int T) {
  const int s = (T + 511) / 512;
  return s < 1 ? 1 : (s > 16 ? 16 : s);
}

cudaError_t attn_decode_launch(const AttnParams& p, cudaStream_t stream, bool pdl) {
  if (p.nsplit > kMaxSplit) return cudaErrorInvalidValue;
  return launch_any(p, 1, stream, pdl);
}

cudaError_t attn_prefill_launch(const AttnParams& p, int M, cudaStream_t stream) {
  if (p.nsplit > kMaxSplit) return cudaErrorInvalidValue;
  return launch_any(p, M, stream, false);
}

}  // namespace sr
