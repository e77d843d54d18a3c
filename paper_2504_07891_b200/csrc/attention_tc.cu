// K4: paged GQA flash attention on the tensor cores (mma.sync m16n8k16, bf16
// in, fp32 accumulate) for the per-kernel decode paths -- the decode graph
// (SR_DECODE=graph, the A/B reference of the persistent kernel) and the
// NCCL tensor-parallel decode loop -- plus the split merge that the prefill
// attention (attention_umma.cu) uses.
//
// Query rows are (token, head-in-group) pairs of one KV head, so the G heads
// sharing a KV head form the MMA's M dimension and every K/V byte is read
// once.  K and V pages (64 positions x 128 dims bf16 = 16 KB each) are staged
// by cp.async into a 2-deep ring with a 16-byte-chunk XOR swizzle so ldmatrix
// is conflict-free; S = Q K^T, an exp2 online softmax in registers, P
// re-packed to bf16 A fragments (FA2-style) and O += P V (ldmatrix.trans on
// V).  A cluster of CTAs splits the KV pages of one kv head and merges
// (m, l, O) through distributed shared memory.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace sr {

constexpr int kTile = kPage;                // 64 positions per KV tile
constexpr int kTileBytes = kTile * kHeadDim * 2;  // 16 KB
constexpr int kAttnMaxSplit = 64;
constexpr float kScaleLog2 = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)

SR_DEV uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

SR_DEV void cpa16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
SR_DEV void cpa_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
SR_DEV void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// swizzled byte offset of (row, 16B-chunk) in a [64][128] bf16 tile
SR_DEV uint32_t swz(int row, int chunk) { return row * 256 + ((chunk ^ (row & 7)) << 4); }

SR_DEV void ldsm4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
SR_DEV void ldsm4t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
SR_DEV void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Per-warp flash state for 16 query rows (thread holds rows g and g+8).
struct Flash {
  float o[16][4];   // 16 dim n-tiles x {row g: c0,c1 ; row g+8: c2,c3}
  float m[2], l[2];
};

// Query row -> (token, head) inside one kv head's group
SR_DEV const __nv_bfloat16* q_row_ptr(const AttnParams& p, int G, int g, int r) {
  const int tok = r / G, j = r % G;
  return p.q + (size_t)tok * p.n_heads * kHeadDim + (size_t)(g * G + j) * kHeadDim;
}

// Split merge for prefill as its own grid-wide kernel: thread = (query row,
// dim); fixed split order (deterministic).  A single last CTA per query tile
// would read every split of 64 rows serially.
__global__ void __launch_bounds__(256) attn_merge_kernel(AttnParams p, int M_rows, int G,
                                                         int nsplit) {
  // warp = one (query row, kv head g); lane = 4 dims.  The (m, l) of all splits
  // are loaded at once (lane sp holds split sp), then every split's 4 dims.
  grid_launch_dependents();
  grid_wait();
  const int g = blockIdx.y, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= M_rows) return;
  constexpr size_t ps = kHeadDim + 2;
  const float* base = p.part + (size_t)g * M_rows * nsplit * ps + (size_t)r * nsplit * ps;
  const float ms = lane < nsplit ? base[lane * ps + kHeadDim] : -INFINITY;
  const float ls = lane < nsplit ? base[lane * ps + kHeadDim + 1] : 0.f;
  float M = ms;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
  float L = w * ls;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  float4 A = make_float4(0.f, 0.f, 0.f, 0.f);
  const int d = 2 * lane;  // dims d, d+1 and 64+d, 64+d+1 (rows are 8-B aligned)
#pragma unroll 4
  for (int sp = 0; sp < nsplit; ++sp) {
    const float ws = __shfl_sync(0xffffffffu, w, sp);
    const float2 a = *reinterpret_cast<const float2*>(base + sp * ps + d);
    const float2 b = *reinterpret_cast<const float2*>(base + sp * ps + 64 + d);
    A.x = fmaf(ws, a.x, A.x);
    A.y = fmaf(ws, a.y, A.y);
    A.z = fmaf(ws, b.x, A.z);
    A.w = fmaf(ws, b.y, A.w);
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  __nv_bfloat16* o = const_cast<__nv_bfloat16*>(q_row_ptr(p, G, g, r)) - p.q + p.out;
  *reinterpret_cast<uint32_t*>(o + d) = f2_to_bf2(A.x * inv, A.y * inv);
  *reinterpret_cast<uint32_t*>(o + 64 + d) = f2_to_bf2(A.z * inv, A.w * inv);
}

cudaError_t attn_merge_launch(const AttnParams& p, int M_tokens, int nsplit, cudaStream_t stream) {
  const int G = p.n_heads / p.n_kv;
  const int M_rows = M_tokens * G;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((M_rows + 7) / 8, p.n_kv);
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_merge_kernel, p, M_rows, G, nsplit);
}

// ----------------------------------------------------------------- decode --
// One cluster of kDecCluster CTAs per KV head; the G query heads of the group
// are the 16-row M tile.  KV tile i (64 positions = one page) belongs to CTA
// i % C.  Inside a CTA all 128 threads stream the CTA's tiles through a
// 2-stage cp.async ring and each warp takes a 16-position quarter of every
// tile (S: 16 HMMA, PV: 32 HMMA with the hi/lo P split), keeping its own
// online-softmax state.  Warps merge (m, l, O) in shared memory; the cluster
// then merges over DSMEM with the work spread across its CTAs (CTA c writes
// dims [16c, 16c + 16)) -- no global partials, no atomics, no extra kernel.
constexpr int kDecCluster = 8;
constexpr int kDecWarps = 4;
constexpr int kDecStages = 2;

struct DecSmem {
  __align__(128) uint8_t k[kDecStages][kTileBytes];
  __align__(128) uint8_t v[kDecStages][kTileBytes];
  __align__(128) uint8_t q[16 * kHeadDim * 2];
  float o[16][kHeadDim];  // CTA-merged, unnormalised O (relative to m)
  float m[16], l[16];
  float wm[kDecWarps][16], wl[kDecWarps][16];
};

// one warp, 16 rows x 16 positions (quarter `sub` of a 64-position tile)
template <bool CAUSAL>
SR_DEV void flash_sub16(Flash& F, const uint32_t (&qa)[8][4], uint32_t ks, uint32_t vs, int lane,
                        int sub, int tile_pos0, int lim) {
  float s[2][4];
#pragma unroll
  for (int n = 0; n < 2; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const int row = sub * 16 + ((lane >> 4) << 3) + (lane & 7);
    const int chunk = kk * 2 + ((lane >> 3) & 1);
    uint32_t b[4];
    ldsm4(b, ks + swz(row, chunk));
    mma_bf16(s[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b[0], b[1]);
    mma_bf16(s[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b[2], b[3]);
  }
  const int t = lane & 3;
  float mx0 = F.m[0], mx1 = F.m[1];
#pragma unroll
  for (int n = 0; n < 2; ++n) {
#pragma unroll
    for (int e = 0; e < 4; ++e) s[n][e] *= kScaleLog2;
    if (CAUSAL) {
      const int p0 = tile_pos0 + sub * 16 + n * 8 + 2 * t;
      if (p0 > lim) { s[n][0] = -INFINITY; s[n][2] = -INFINITY; }
      if (p0 + 1 > lim) { s[n][1] = -INFINITY; s[n][3] = -INFINITY; }
    }
    mx0 = fmaxf(mx0, fmaxf(s[n][0], s[n][1]));
    mx1 = fmaxf(mx1, fmaxf(s[n][2], s[n][3]));
  }
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
  mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
  mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
  const float base0 = mx0 == -INFINITY ? 0.f : mx0;
  const float base1 = mx1 == -INFINITY ? 0.f : mx1;
  const float c0 = exp2f(F.m[0] - base0), c1 = exp2f(F.m[1] - base1);
  F.m[0] = mx0;
  F.m[1] = mx1;
  float rs0 = 0.f, rs1 = 0.f;
  uint32_t pa[4], pl[4];
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    const float e0 = exp2f(s[n][0] - base0), e1 = exp2f(s[n][1] - base0);
    const float e2 = exp2f(s[n][2] - base1), e3 = exp2f(s[n][3] - base1);
    rs0 += e0 + e1;
    rs1 += e2 + e3;
    const uint32_t h01 = f2_to_bf2(e0, e1), h23 = f2_to_bf2(e2, e3);
    const float2 r01 = bf2_to_f2(h01), r23 = bf2_to_f2(h23);
    pa[2 * n] = h01;
    pa[2 * n + 1] = h23;
    pl[2 * n] = f2_to_bf2(e0 - r01.x, e1 - r01.y);
    pl[2 * n + 1] = f2_to_bf2(e2 - r23.x, e3 - r23.y);
  }
  F.l[0] = F.l[0] * c0 + rs0;
  F.l[1] = F.l[1] * c1 + rs1;
#pragma unroll
  for (int d = 0; d < 16; ++d) {
    F.o[d][0] *= c0; F.o[d][1] *= c0;
    F.o[d][2] *= c1; F.o[d][3] *= c1;
  }
#pragma unroll
  for (int dp = 0; dp < 8; ++dp) {
    const int row = sub * 16 + (((lane >> 3) & 1) << 3) + (lane & 7);
    const int chunk = dp * 2 + (lane >> 4);
    uint32_t b[4];
    ldsm4t(b, vs + swz(row, chunk));
    mma_bf16(F.o[2 * dp], pa[0], pa[1], pa[2], pa[3], b[0], b[1]);
    mma_bf16(F.o[2 * dp + 1], pa[0], pa[1], pa[2], pa[3], b[2], b[3]);
    mma_bf16(F.o[2 * dp], pl[0], pl[1], pl[2], pl[3], b[0], b[1]);
    mma_bf16(F.o[2 * dp + 1], pl[0], pl[1], pl[2], pl[3], b[2], b[3]);
  }
}

__global__ void __cluster_dims__(1, kDecCluster, 1) __launch_bounds__(kDecWarps * 32)
    attn_decode_tc_kernel(AttnParams p, int G) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  DecSmem& sm = *reinterpret_cast<DecSmem*>(smem_raw);
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();

  grid_launch_dependents();
  grid_wait();
  const bool done = p.st->done != 0;  // same for every CTA of the launch

  const int g = blockIdx.x;
  const int crank = (int)cluster.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2;

  Flash F;
#pragma unroll
  for (int d = 0; d < 16; ++d) F.o[d][0] = F.o[d][1] = F.o[d][2] = F.o[d][3] = 0.f;
  F.m[0] = F.m[1] = -INFINITY;
  F.l[0] = F.l[1] = 0.f;

  if (!done) {
    const int T = p.st->ctx_len;
    const int* ptab = p.st->page_table;
    const int n_tiles = (T + kTile - 1) / kTile;
    const int n_mine = n_tiles > crank ? (n_tiles - crank + kDecCluster - 1) / kDecCluster : 0;
    auto issue = [&](int j, int stage) {
      const int i = crank + j * kDecCluster;
      const size_t off = kv_offset(p.layer, ptab[i], g, 0, p.n_pages, p.n_kv);
      const uint8_t* kg = reinterpret_cast<const uint8_t*>(p.k_pool + off);
      const uint8_t* vg = reinterpret_cast<const uint8_t*>(p.v_pool + off);
      const uint32_t kb = s_u32(sm.k[stage]), vb = s_u32(sm.v[stage]);
#pragma unroll
      for (int c = tid; c < kTile * 16; c += kDecWarps * 32) {
        const int r = c >> 4, ch = c & 15;
        cpa16(kb + swz(r, ch), kg + r * 256 + ch * 16);
        cpa16(vb + swz(r, ch), vg + r * 256 + ch * 16);
      }
    };
    if (n_mine > 0) issue(0, 0);
    cpa_commit();
    for (int i = tid; i < 16 * 16; i += kDecWarps * 32) {
      const int r = i >> 4, c = i & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < G) v = reinterpret_cast<const uint4*>(p.q + (size_t)(g * G + r) * kHeadDim)[c];
      *reinterpret_cast<uint4*>(sm.q + swz(r, c)) = v;
    }
    __syncthreads();
    uint32_t qa[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) ldsm4(qa[kk], s_u32(sm.q) + swz(lane & 15, kk * 2 + (lane >> 4)));
    const int lim = T - 1;
    for (int j = 0; j < n_mine; ++j) {
      const int stage = j & 1;
      if (j + 1 < n_mine) issue(j + 1, stage ^ 1);
      cpa_commit();
      cpa_wait<1>();
      __syncthreads();
      const int pos0 = (crank + j * kDecCluster) * kTile;
      const uint32_t ks = s_u32(sm.k[stage]), vs = s_u32(sm.v[stage]);
      if (pos0 + kTile - 1 > lim) flash_sub16<true>(F, qa, ks, vs, lane, warp, pos0, lim);
      else flash_sub16<false>(F, qa, ks, vs, lane, warp, pos0, lim);
      __syncthreads();
    }
    cpa_wait<0>();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      F.l[h] += __shfl_xor_sync(0xffffffffu, F.l[h], 1);
      F.l[h] += __shfl_xor_sync(0xffffffffu, F.l[h], 2);
    }
  }

  // ---- merge the 4 warps of this CTA (fixed order: deterministic) ----
  if ((lane & 3) == 0) {
    sm.wm[warp][gq] = F.m[0];
    sm.wm[warp][gq + 8] = F.m[1];
    sm.wl[warp][gq] = F.l[0];
    sm.wl[warp][gq + 8] = F.l[1];
  }
  for (int i = tid; i < 16 * kHeadDim; i += kDecWarps * 32) (&sm.o[0][0])[i] = 0.f;
  __syncthreads();
  if (tid < 16) {
    float M = -INFINITY, L = 0.f;
    for (int w = 0; w < kDecWarps; ++w) M = fmaxf(M, sm.wm[w][tid]);
    for (int w = 0; w < kDecWarps; ++w) {
      const float mw = sm.wm[w][tid];
      L += mw == -INFINITY ? 0.f : sm.wl[w][tid] * exp2f(mw - M);
    }
    sm.m[tid] = M;
    sm.l[tid] = L;
  }
  __syncthreads();
  for (int w = 0; w < kDecWarps; ++w) {
    if (w == warp) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = gq + 8 * h;
        const float mw = F.m[h], M = sm.m[rr];
        const float c = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
#pragma unroll
        for (int d = 0; d < 16; ++d) {
          const int col = d * 8 + 2 * (lane & 3);
          sm.o[rr][col] += F.o[d][2 * h] * c;
          sm.o[rr][col + 1] += F.o[d][2 * h + 1] * c;
        }
      }
    }
    __syncthreads();
  }

  // ---- cluster merge over DSMEM, spread over the CTAs: CTA c writes dims [16c, 16c+16) ----
  cluster.sync();
  if (!done) {
    constexpr int kDims = kHeadDim / kDecCluster;
    for (int idx = tid; idx < G * kDims; idx += kDecWarps * 32) {
      const int rr = idx / kDims, d = crank * kDims + idx % kDims;
      float mc[kDecCluster];
      float M = -INFINITY;
#pragma unroll
      for (int c = 0; c < kDecCluster; ++c) {
        mc[c] = cluster.map_shared_rank(&sm, c)->m[rr];
        M = fmaxf(M, mc[c]);
      }
      float L = 0.f, A = 0.f;
#pragma unroll
      for (int c = 0; c < kDecCluster; ++c) {
        if (mc[c] == -INFINITY) continue;
        const DecSmem* r = cluster.map_shared_rank(&sm, c);
        const float w = exp2f(mc[c] - M);
        L += r->l[rr] * w;
        A += r->o[rr][d] * w;
      }
      p.out[(size_t)(g * G + rr) * kHeadDim + d] = __float2bfloat16_rn(L > 0.f ? A / L : 0.f);
    }
  }
  cluster.sync();  // keep every CTA's shared memory alive until all reads are done
}

cudaError_t attn_decode_tc_launch(const AttnParams& p, cudaStream_t stream, bool pdl) {
  const int G = p.n_heads / p.n_kv;
  if (G > 16) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_decode_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(DecSmem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_kv, kDecCluster, 1);
  cfg.blockDim = dim3(kDecWarps * 32);
  cfg.dynamicSmemBytes = sizeof(DecSmem);
  cfg.stream = stream;
  cudaLaunchAttribute attr_l[1];
  attr_l[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr_l[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr_l;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_decode_tc_kernel, p, G);
}

// decode attention splits per kv head: ~one CTA per SM at long contexts
int attn_decode_splits(int n_kv, int num_sms) {
  int s = (num_sms + n_kv - 1) / n_kv;
  return s < 1 ? 1 : (s > kAttnMaxSplit ? kAttnMaxSplit : s);
}

}  // namespace sr
