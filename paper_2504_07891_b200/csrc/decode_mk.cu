// Persistent weight-streaming decode kernel: K1 + K3 + K4 + K5 + K10 fused.
//
// One launch decodes a whole reasoning step (every token until a stop-class
// token, </think> or max_new).  One CTA per SM (grid = #SMs, cooperative
// launch so all CTAs are co-resident); each CTA has
//
//   * a producer warp: one lane streams the CTA's share of every weight matrix
//     of the model -- layer 0 qkv, o, gate/up, down, layer 1 ..., LM head, then
//     the next token's layer 0 ... -- as 32-row x 256-column bf16 tiles (16 KB)
//     into an mbarrier ring of up to 13 stages (2 tiles each).  Default
//     (kTiled): from the tile-major, pre-swizzled copy of the weights
//     (sr_model_set_decode_tiles), one contiguous 16 KB cp.async.bulk per
//     tile; else (SR_MK_TILED=0) a TMA box of the row-major weights.  Weights
//     are constant, so the producer never waits for activations: it runs
//     ahead across phase and grid barriers and into the next token, bounded
//     only by the ring;
//   * 16 consumer warps that run the token's phases in order, separated by
//     grid barriers (one atomic counter, acquire/release):
//
//       per layer: QKV | ATTN | COMBINE | O | GATE/UP | DOWN      then: LM head
//
// GEMV phases.  A phase's tiles ("units", row-block major, k minor) are cut
// into G contiguous ranges, one per CTA, so every CTA streams the same number
// of bytes (+-1 tile).  Tensor-core consumer (mk_gemv_mma, default): warp w
// takes rows 16(w&1).. and columns 32(w>>1).. of every tile with two
// mma.sync m16n8k16 (x as every column of B), accumulating over the k tiles
// of a row block; at its end the 8 column slices of each row are summed in
// fixed order through shared memory.  CUDA-core consumer (mk_gemv): warp w
// owns rows w and w+16, lane = 8 columns.  A row block cut by a range
// boundary leaves one partial per contributing CTA in `part[cta][j][32]`;
// the next phase's prologue sums the partials of each row in CTA order
// (deterministic, no atomics).  GATE/UP and LM head use block-granular ranges
// instead: the interleaved gate/up layout (16 gate rows then the 16 matching
// up rows per 32-row block) lets the gate/up epilogue emit silu(g)*u
// directly, and the LM head needs whole logits for the greedy argmax.
//
// Prologues.  Every CTA rebuilds the GEMV input vector x in shared memory:
// RMSNorm(h) from the fp32 residual stream plus the previous phase's partials
// (16-B loads, one batch; CTA 0 writes the updated residual back; two buffers
// alternate so no CTA reads a vector while it is rewritten), or a copy of the
// bf16 attention output / activation.  All cross-CTA data is read with
// ld.global.cg (L2), never through the non-coherent L1.
//
// Attention (K4).  CTA (kv head g, split s) takes a contiguous page range of
// the paged K/V cache for the query heads of g: q and the new k/v are summed
// from the qkv partials (+bias, RoPE, bf16 rounding as the oracle), the CTA
// owning the last page appends k/v to the pool.  Pages arrive as 128-B-
// swizzled TMA boxes; S = Q.K^T and O += P.V run on mma.sync with an exp2
// online softmax in between (P as bf16 hi + lo), pipelined over two warp
// groups where a second page buffer fits.  COMBINE merges the split partials
// per head into the bf16 attention output.
//
// LM head (K5).  Each CTA keeps a (top-1, index, top-2) over its rows; after
// the barrier every CTA merges the G partials (ties -> lower index), so all of
// them agree on the token and on `done` without another barrier; CTA 0 writes
// the token, margin and stop state exactly as select_token() does.
#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace sr {

#ifndef SR_MK_WARPS
#define SR_MK_WARPS 16
#endif
constexpr int kMkWarps = SR_MK_WARPS;      // consumer warps (16 or 8)
constexpr int kMkConsumers = kMkWarps * 32;
constexpr int kRW = 32 / kMkWarps;          // rows of a 32-row tile per warp
static_assert(kMkWarps == 16, "attention: warp w owns head dims 8w..8w+7 of P.V");
constexpr int kMkThreads = kMkConsumers + 32;
constexpr int kTR = 32;                    // tile rows
constexpr int kTC = 256;                   // tile columns (bf16)
constexpr int kTileBytes = kTR * kTC * 2;  // 16 KB
constexpr int kSubTileBytes = kTR * 64 * 2; // one [32][64] swizzled box of a tile-major tile (4 KB)
#ifndef SR_MK_NB
#define SR_MK_NB 4
#endif
#ifndef SR_MK_UPS
#define SR_MK_UPS 2
#endif
constexpr int kUPS = SR_MK_UPS;            // tiles ("units") per ring stage
constexpr int kStageBytes = kUPS * kTileBytes;
constexpr int kMkMaxStages = 13;
constexpr int kMkMaxGq = 8;
constexpr int kMkProfEvents = SR_PROF_EVENTS;
constexpr int kMkAttnScratchFloats = 2048;  // attention q / P / row partials; COMBINE [16][64]+32
constexpr int kMkTab = 256;  // max 32-row blocks of a tile-range phase (smem tables)
constexpr int kKvBufBytes = 2 * kPage * kHeadDim * 2;  // K + V page (32 KB)

enum { PH_QKV = 0, PH_O = 1, PH_GU = 2, PH_D = 3, PH_LM = 4 };

struct Geo {
  int tc, kt, nb, T, blockpart;  // tile columns (256, or K when K < 256), k tiles, row blocks, units
};

SR_DEV Geo mk_geo(const MkParams& p, int ph) {
  int N, K;
  switch (ph) {
    case PH_QKV: N = p.qkv_rows; K = p.d; break;
    case PH_O: N = p.d; K = p.q_dim; break;
    case PH_GU: N = 2 * p.f; K = p.d; break;
    case PH_D: N = p.d; K = p.f; break;
    default: N = p.vocab_rows; K = p.d; break;
  }
  Geo g;
  g.tc = K < kTC ? K : kTC;
  g.kt = (K + g.tc - 1) / g.tc;
  g.nb = (N + kTR - 1) / kTR;
  g.T = g.nb * g.kt;
  g.blockpart = (ph == PH_GU || ph == PH_LM);
  return g;
}

SR_DEV void mk_range(const Geo& g, int c, int G, int& lo, int& hi) {
  if (g.blockpart) {
    lo = (int)((long long)g.nb * c / G) * g.kt;
    hi = (int)((long long)g.nb * (c + 1) / G) * g.kt;
  } else if (g.T >= G) {
    lo = (int)((long long)g.T * c / G);
    hi = (int)((long long)g.T * (c + 1) / G);
  } else {  // fewer tiles than CTAs: one tile each for the first T CTAs
    lo = c < g.T ? c : g.T;
    hi = c < g.T ? c + 1 : g.T;
  }
}

// this CTA's tile range of one phase, precomputed once per launch (no integer
// division on the per-tile paths)
struct PhaseInfo {
  int lo, hi;    // unit range
  int kt, tc;    // k tiles per row block, tile columns
  int b0, k0;    // row block / k tile of unit lo
  int bytes;     // bytes per tile
  int pad;
};

SR_DEV PhaseInfo mk_phase_info(const MkParams& p, int ph, int c, int G) {
  const Geo g = mk_geo(p, ph);
  PhaseInfo pi;
  mk_range(g, c, G, pi.lo, pi.hi);
  pi.kt = g.kt;
  pi.tc = g.tc;
  pi.b0 = pi.lo / g.kt;
  pi.k0 = pi.lo - pi.b0 * g.kt;
  pi.bytes = kTR * g.tc * 2;
  pi.pad = 0;
  return pi;
}

// sum of the partials of `row` left by a tile-range phase, in CTA order
// (deterministic).  tab[block] = {first contributing CTA, #contributors, slot j
// of the block in the first CTA's range}; later contributors hold it at j = 0.
// (packed in shared memory as c0 | n << 8 | j0 << 12)
SR_DEV float mk_sum_parts(const float* part, const uint16_t* tab, int row, int maxj) {
  const int b = row / kTR, r = row % kTR;
  const int e = tab[b];
  const int c0 = e & 0xff, n = (e >> 8) & 0xf, j0 = e >> 12;
  const size_t cs = (size_t)maxj * kTR;
  const float* q1 = part + (size_t)(c0 + 1) * cs + r;
  // up to eight contributors as independent predicated loads, all in flight
  // together (no loop: the unrolled callers keep every row's loads batched)
  float a[8];
  a[0] = __ldcg(part + (size_t)c0 * cs + (size_t)j0 * kTR + r);
#pragma unroll
  for (int q = 1; q < 8; ++q) a[q] = n > q ? __ldcg(q1 + (size_t)(q - 1) * cs) : 0.f;
  float s = a[0];
#pragma unroll
  for (int q = 1; q < 8; ++q) s += a[q];
  return s;
}

SR_DEV void cbar() { asm volatile("bar.sync 1, %0;" ::"n"(kMkConsumers) : "memory"); }

SR_DEV float cblock_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[w] = v;
  cbar();
  float t = lane < kMkWarps ? red[lane] : 0.f;
  t = warp_sum(t);
  cbar();
  return t;
}

SR_DEV uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// grid barrier over the consumer threads of all CTAs: the CTA barrier orders
// every consumer's writes before thread 0's release-add; thread 0's acquire
// poll + the CTA barrier order them before every consumer's later reads
SR_DEV void mk_grid_sync(unsigned* ctr, unsigned& target, int G, int sleep_ns) {
  cbar();
  target += (unsigned)G;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    const uint64_t t0 = global_ns();
    for (unsigned spin = 0;; ++spin) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      if (sleep_ns > 0) __nanosleep(sleep_ns);
      if ((spin & 1023) == 1023 && global_ns() - t0 > 5000000000ull) __trap();
    }
  }
  cbar();
}

// x = bf16(h * rstd * w) with h = embedding row (mode 0) or hin + partials;
// zero padding up to the next multiple of 256; CTA 0 stores h to hout.
// Rows are processed in batches: every load of a batch (residual, norm
// weight, up to four partials per row) is issued before any is used, so a
// batch costs one round trip; h and w wait in shared memory (`tmp`, the idle
// K/V page buffer) for the block-wide sum of squares.
// With tensor parallelism (`mb` non-null, mode 1) the update is instead the
// all-ranks sum read from this rank's decode mailbox: h = hin + sum over
// ranks q = 0..W-1 (in rank order) of mb[q][i].
SR_DEV void mk_norm_prologue(const MkParams& p, int mode, int tok, const float* hin,
                             const float* part, const uint16_t* tab, const __nv_bfloat16* w,
                             float* hout, __nv_bfloat16* xs, float* red, int c, int G,
                             float* tmp, const float* mb = nullptr, int prof_slot = -1) {
  const int d = p.d, tid = threadIdx.x;
  const bool pe = prof_slot >= 0 && p.prof && c == 0 && tid == 0;
  if (pe) p.prof[prof_slot] = global_ns();
  float* hs = tmp;                                            // [d] fp32
  __nv_bfloat16* wsm = reinterpret_cast<__nv_bfloat16*>(tmp + d);  // [d] bf16
  float ss = 0.f;
  constexpr int kNB = SR_MK_NB;  // rows per thread per load batch
  const size_t cs = (size_t)p.maxj * kTR;
  if (mode == 1 && !mb && p.vec_prologue) {
    // residual + split partials, 4 rows per 16-B load: up to 3 x 512 groups
    // (d <= 6144) in one batch, i.e. one L2 round trip (rows cut over more
    // than two CTAs -- small models only -- add a second)
    constexpr int kG = 3;
    const int ng = d / 4;
#pragma unroll 1
    for (int g0 = tid; g0 < ng; g0 += kG * kMkConsumers) {
      float4 hb[kG], pa[kG], pq[kG];
      uint2 wb[kG];
      int nv[kG];
#pragma unroll
      for (int jj = 0; jj < kG; ++jj) {
        const int gi = g0 + jj * kMkConsumers;
        const int i = (gi < ng ? gi : 0) * 4;
        wb[jj] = *reinterpret_cast<const uint2*>(w + i);
        hb[jj] = __ldcg(reinterpret_cast<const float4*>(hin + i));
        const int e = tab[i / kTR], r = i % kTR;
        const int c0 = e & 0xff, n = (e >> 8) & 0xf, j0 = e >> 12;
        pa[jj] = __ldcg(reinterpret_cast<const float4*>(part + (size_t)c0 * cs + (size_t)j0 * kTR + r));
        pq[jj] = n > 1 ? __ldcg(reinterpret_cast<const float4*>(part + (size_t)(c0 + 1) * cs + r))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        nv[jj] = gi < ng ? n : 0;
      }
#pragma unroll
      for (int jj = 0; jj < kG; ++jj) {
        if (nv[jj] == 0) continue;
        const int i = (g0 + jj * kMkConsumers) * 4;
        float4 sp = make_float4(pa[jj].x + pq[jj].x, pa[jj].y + pq[jj].y, pa[jj].z + pq[jj].z,
                                pa[jj].w + pq[jj].w);
        if (nv[jj] > 2) {
          const int c0 = tab[i / kTR] & 0xff, r = i % kTR;
          for (int q = 2; q < nv[jj]; ++q) {
            const float4 t = __ldcg(reinterpret_cast<const float4*>(part + (size_t)(c0 + q) * cs + r));
            sp.x += t.x;
            sp.y += t.y;
            sp.z += t.z;
            sp.w += t.w;
          }
        }
        const float4 v = make_float4(hb[jj].x + sp.x, hb[jj].y + sp.y, hb[jj].z + sp.z, hb[jj].w + sp.w);
        *reinterpret_cast<float4*>(hs + i) = v;
        *reinterpret_cast<uint2*>(wsm + i) = wb[jj];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
      }
    }
  } else
#pragma unroll 1
  for (int i0 = tid; i0 < d; i0 += kNB * kMkConsumers) {
    float hb[kNB], pb[kNB][4];
    __nv_bfloat16 wb[kNB];
    int nb[kNB];
#pragma unroll
    for (int jj = 0; jj < kNB; ++jj) {
      const int i = i0 + jj * kMkConsumers;
      const bool ok = i < d;
      const int ic = ok ? i : 0;
      wb[jj] = w[ic];
      if (mode == 0) {
        hb[jj] = bf_to_f(p.embed[(size_t)tok * d + ic]);
        nb[jj] = 0;
        pb[jj][0] = pb[jj][1] = pb[jj][2] = pb[jj][3] = 0.f;
      } else if (mb) {  // tensor parallel: the ranks' deltas, summed in rank order
        hb[jj] = __ldcg(hin + ic);
        float r[kPeerMaxWorld];
#pragma unroll
        for (int q = 0; q < kPeerMaxWorld; ++q)
          r[q] = q < p.tp_world ? __ldcg(mb + (size_t)q * p.tp_dec_row + ic) : 0.f;
        float sp = r[0];
#pragma unroll
        for (int q = 1; q < kPeerMaxWorld; ++q) sp += r[q];
        pb[jj][0] = sp;
        pb[jj][1] = pb[jj][2] = pb[jj][3] = 0.f;
        nb[jj] = 1;
      } else {
        hb[jj] = __ldcg(hin + ic);
        const int e = tab[ic / kTR];
        const int r = ic % kTR;
        const int c0 = e & 0xff, n = (e >> 8) & 0xf, jo = e >> 12;
        const float* q1 = part + (size_t)(c0 + 1) * cs + r;
        pb[jj][0] = __ldcg(part + (size_t)c0 * cs + (size_t)jo * kTR + r);
        pb[jj][1] = n > 1 ? __ldcg(q1) : 0.f;
        pb[jj][2] = n > 2 ? __ldcg(q1 + cs) : 0.f;
        pb[jj][3] = n > 3 ? __ldcg(q1 + 2 * cs) : 0.f;
        nb[jj] = n;
      }
    }
#pragma unroll
    for (int jj = 0; jj < kNB; ++jj) {
      const int i = i0 + jj * kMkConsumers;
      if (i < d) {
        float v = hb[jj];
        if (mode != 0) {
          float sp = ((pb[jj][0] + pb[jj][1]) + pb[jj][2]) + pb[jj][3];
          if (nb[jj] > 4) {  // tiny models only: more contributors than a batch holds
            const int e = tab[i / kTR];
            for (int q = 4; q < nb[jj]; ++q)
              sp += __ldcg(part + (size_t)((e & 0xff) + q) * cs + i % kTR);
          }
          v += sp;
        }
        hs[i] = v;
        wsm[i] = wb[jj];
        ss += v * v;
      }
    }
  }
  if (pe) p.prof[prof_slot + 1] = global_ns();
  ss = cblock_sum(ss, red);  // (its barriers also publish hs / wsm)
  if (pe) p.prof[prof_slot + 2] = global_ns();
  const float rstd = rsqrtf(ss / d + p.eps);
  const int dpad = (d + kTC - 1) / kTC * kTC;
  for (int i = tid; i < d; i += kMkConsumers) {
    const float v = hs[i];
    xs[i] = __float2bfloat16_rn(v * rstd * bf_to_f(wsm[i]));
    if (c == 0 && hout) hout[i] = v;
  }
  for (int i = d + tid; i < dpad; i += kMkConsumers) xs[i] = __float2bfloat16_rn(0.f);
  cbar();
  if (pe) p.prof[prof_slot + 3] = global_ns();
}

SR_DEV void mk_stage_vec(const __nv_bfloat16* src, int K, __nv_bfloat16* xs) {
  const int Kp = (K + kTC - 1) / kTC * kTC;
  for (int i = threadIdx.x; i < K / 8; i += kMkConsumers) {
    uint4 v = __ldcg(reinterpret_cast<const uint4*>(src) + i);
    reinterpret_cast<uint4*>(xs)[i] = v;
  }
  for (int i = K + threadIdx.x; i < Kp; i += kMkConsumers) xs[i] = __float2bfloat16_rn(0.f);
  cbar();
}

// Tensor parallelism: after a row-parallel phase (O, down) and its grid
// barrier, CTA c sums this rank's split partials of rows [c*d/G, (c+1)*d/G)
// (the rank's delta) and stores them into slot [rank] of every rank's decode
// mailbox over NVLink; thread 0 then release-adds every rank's flag and
// acquires its own until all W*G arrivals of this exchange are in.  Returns
// this rank's mailbox slot, which the next prologue sums in rank order.
SR_DEV const float* mk_tp_exchange(const MkParams& p, const float* part, const uint16_t* tab,
                                   unsigned& ex, int c, int G) {
  const int slot = (int)(ex & 1u);
  const unsigned target = (ex / 2 + 1) * (unsigned)(p.tp_world * G);
  ex += 1;
  const size_t soff = p.tp_off_dec + (size_t)slot * p.tp_world * p.tp_dec_row * 4;
  const int r0 = (int)((long long)p.d * c / G), r1 = (int)((long long)p.d * (c + 1) / G);
  for (int i = r0 + (int)threadIdx.x; i < r1; i += kMkConsumers) {
    const float v = mk_sum_parts(part, tab, i, p.maxj);
    for (int q = 0; q < p.tp_world; ++q)
      reinterpret_cast<float*>(p.tp_base[q] + soff)[(size_t)p.tp_rank * p.tp_dec_row + i] = v;
  }
  cbar();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < p.tp_world; ++q)
      red_release_sys(reinterpret_cast<unsigned*>(p.tp_base[q]) + 2 + slot, 1u);
    peer_wait(reinterpret_cast<const unsigned*>(p.tp_base[p.tp_rank]) + 2 + slot, target);
  }
  cbar();
  return reinterpret_cast<const float*>(p.tp_base[p.tp_rank] + soff);
}

// Tensor parallelism: the vocab-parallel greedy merge.  Every CTA holds this
// rank's (top-1, global index, top-2); CTA 0 stores it into slot [rank] of
// every rank's greedy mailbox; all CTAs wait for the W entries and merge them
// in rank order (ties -> lower id), so every rank picks the same token.
SR_DEV Top2 mk_tp_merge(const MkParams& p, Top2 mine, unsigned& lx, int c) {
  const int slot = (int)(lx & 1u);
  const unsigned target = (lx / 2 + 1) * (unsigned)p.tp_world;
  lx += 1;
  const size_t soff = p.tp_off_lm + (size_t)slot * p.tp_world * 4 * 4;
  if (c == 0 && threadIdx.x == 0) {
    for (int q = 0; q < p.tp_world; ++q) {
      float* dst = reinterpret_cast<float*>(p.tp_base[q] + soff) + p.tp_rank * 4;
      dst[0] = mine.v1;
      dst[1] = __int_as_float(mine.i1);
      dst[2] = mine.v2;
    }
    __threadfence_system();
    for (int q = 0; q < p.tp_world; ++q)
      red_release_sys(reinterpret_cast<unsigned*>(p.tp_base[q]) + 4 + slot, 1u);
  }
  __shared__ float s_m[kPeerMaxWorld * 4];
  if (threadIdx.x == 0) {
    peer_wait(reinterpret_cast<const unsigned*>(p.tp_base[p.tp_rank]) + 4 + slot, target);
    const float* mb = reinterpret_cast<const float*>(p.tp_base[p.tp_rank] + soff);
    for (int i = 0; i < 4 * p.tp_world; ++i) s_m[i] = __ldcg(mb + i);
  }
  cbar();
  Top2 b;
  b.init();
  for (int q = 0; q < p.tp_world; ++q) b.merge(s_m[4 * q], __float_as_int(s_m[4 * q + 1]), s_m[4 * q + 2]);
  cbar();
  return b;
}

// ring position shared by the consumer warps (every warp walks every stage)
struct RingPos {
  int slot;
  uint32_t par;
  SR_DEV void advance(int S) {
    if (++slot == S) {
      slot = 0;
      par ^= 1u;
    }
  }
};

// consume this CTA's tiles of one GEMV phase (same order as the producer):
// a ring stage carries up to kUPS consecutive tiles of the phase, so the
// per-stage handshake (wait, arrive) is paid once per kUPS x 16 KB
template <int PH>
SR_DEV void mk_gemv(const MkParams& p, const PhaseInfo& pi, int c, const uint8_t* ring,
                    uint64_t* full, uint64_t* empty, const __nv_bfloat16* xs, RingPos& rp, int S,
                    Top2& best) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lo = pi.lo, hi = pi.hi, kt = pi.kt, tc = pi.tc;
  const int row_bytes = tc * 2;
  const bool active = lane * 8 < tc;
  int b = pi.b0, k = pi.k0;
  float a[kRW];
#pragma unroll
  for (int i = 0; i < kRW; ++i) a[i] = 0.f;
  for (int u0 = lo; u0 < hi; u0 += kUPS) {
    mbar_wait(&full[rp.slot], rp.par);
    const uint8_t* stage = ring + (size_t)rp.slot * kStageBytes;
    const int nu = hi - u0 < kUPS ? hi - u0 : kUPS;
#pragma unroll
    for (int q = 0; q < kUPS; ++q) {
      if (q < nu) {
        const int u = u0 + q;
        if (active) {
          const uint8_t* tile = stage + q * kTileBytes;
          const uint4 xv = *reinterpret_cast<const uint4*>(xs + k * tc + lane * 8);
#pragma unroll
          for (int i = 0; i < kRW; ++i) {
            const uint4 w = *reinterpret_cast<const uint4*>(tile + (warp + i * kMkWarps) * row_bytes + lane * 16);
            a[i] = dot8(w, xv, a[i]);
          }
        }
        if (q == nu - 1) {  // stage fully read: hand it back to the producer
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[rp.slot]);
          rp.advance(S);
        }
        if (k == kt - 1 || u == hi - 1) {
#pragma unroll
          for (int i = 0; i < kRW; ++i) a[i] = warp_sum(a[i]);
          if (lane == 0) {
            if constexpr (PH == PH_QKV || PH == PH_O || PH == PH_D) {
              float* part = PH == PH_QKV ? p.part_qkv : PH == PH_O ? p.part_o : p.part_d;
              float* dst = part + ((size_t)c * p.maxj + (b - pi.b0)) * kTR;
#pragma unroll
              for (int i = 0; i < kRW; ++i) dst[warp + i * kMkWarps] = a[i];
            } else if constexpr (PH == PH_GU) {
              // rows warp + i*W (< 16) are gate units, +16 their up rows
#pragma unroll
              for (int i = 0; i < kRW / 2; ++i) {
                const float g = a[i], up = a[i + kRW / 2];
                p.act[b * 16 + warp + i * kMkWarps] = __float2bfloat16_rn(g / (1.f + __expf(-g)) * up);
              }
            } else {
#pragma unroll
              for (int i = 0; i < kRW; ++i) {
                const int r = b * kTR + warp + i * kMkWarps;
                if (r < p.vocab_text) best.push(a[i], r);
              }
            }
          }
#pragma unroll
          for (int i = 0; i < kRW; ++i) a[i] = 0.f;
        }
        if (++k == kt) {
          k = 0;
          ++b;
        }
      }
    }
  }
}


// Tensor-core form of mk_gemv (p.tiled): the tile arrives (one bulk copy of
// the tile-major weights) as tc/64 boxes of 32 rows x 64 columns, 128-B swizzled (16-B chunk j of row r at
// r * 128 + ((j ^ (r & 7)) << 4)).  Warp w owns rows 16*(w & 1) .. +15 and
// columns 32*(w >> 1) .. +31 of every tile: two m16n8k16 MMAs per tile with
// the weights as A (ldmatrix.x4) and x as every column of B, so each of the
// 8 output columns is the same dot product.  The fp32 accumulators run over
// the row block's k tiles; at its end the 8 column slices of each row are
// summed in fixed order through shared memory (one barrier per row block,
// double-buffered) and thread r < 32 finishes row r exactly as mk_gemv does.
SR_DEV void mma16816f(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int PH>
SR_DEV void mk_gemv_mma(const MkParams& p, const PhaseInfo& pi, int c, const uint8_t* ring,
                        uint64_t* full, uint64_t* empty, const __nv_bfloat16* xs, RingPos& rp, int S,
                        Top2& best, float* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lo = pi.lo, hi = pi.hi, kt = pi.kt, tc = pi.tc;
  const int mt = warp & 1, ks = warp >> 1;           // row half, 32-column slice
  const bool active = 32 * ks < tc;
  const int r16 = 16 * mt + (lane & 15);              // A row this lane addresses
  const int sub = ks >> 1, ch0 = (ks & 1) * 4 + (lane >> 4);
  // byte offset in a tile of (row r16, chunk ch0 + 2 * step) for steps 0, 1
  const uint32_t a_off0 = sub * kSubTileBytes + r16 * 128 + (((ch0) ^ (r16 & 7)) << 4);
  const uint32_t a_off1 = sub * kSubTileBytes + r16 * 128 + (((ch0 + 2) ^ (r16 & 7)) << 4);
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t xs_s = smem_u32(xs) + (32 * ks + 2 * (lane & 3)) * 2;
  const int g = lane >> 2;
  int b = pi.b0, k = pi.k0, blk = 0;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int u0 = lo; u0 < hi; u0 += kUPS) {
    mbar_wait(&full[rp.slot], rp.par);
    const uint32_t stage = ring_s + rp.slot * kStageBytes;
    const int nu = hi - u0 < kUPS ? hi - u0 : kUPS;
#pragma unroll
    for (int q = 0; q < kUPS; ++q) {
      if (q < nu) {
        const int u = u0 + q;
        if (active) {
          const uint32_t t = stage + q * kTileBytes;
          uint32_t a0[4], a1[4], x0, x1, x2, x3;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(a0[0]), "=r"(a0[1]), "=r"(a0[2]), "=r"(a0[3]) : "r"(t + a_off0));
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(a1[0]), "=r"(a1[1]), "=r"(a1[2]), "=r"(a1[3]) : "r"(t + a_off1));
          const uint32_t xa = xs_s + k * tc * 2;
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x0) : "r"(xa));
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x1) : "r"(xa + 16));
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x2) : "r"(xa + 32));
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x3) : "r"(xa + 48));
          mma16816f(acc, a0, x0, x1);
          mma16816f(acc, a1, x2, x3);
        }
        if (q == nu - 1) {  // stage fully read: hand it back to the producer
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[rp.slot]);
          rp.advance(S);
        }
        if (k == kt - 1 || u == hi - 1) {
          float* rb = red + (blk & 1) * 256;  // [8 slices][32 rows]
          if ((lane & 3) == 0) {
            rb[ks * 32 + 16 * mt + g] = acc[0];
            rb[ks * 32 + 16 * mt + g + 8] = acc[2];
          }
          cbar();
          if (warp == 0) {
            float v = rb[lane];
#pragma unroll
            for (int s2 = 1; s2 < 8; ++s2) v += rb[s2 * 32 + lane];
            if constexpr (PH == PH_QKV || PH == PH_O || PH == PH_D) {
              float* part = PH == PH_QKV ? p.part_qkv : PH == PH_O ? p.part_o : p.part_d;
              part[((size_t)c * p.maxj + (b - pi.b0)) * kTR + lane] = v;
            } else if constexpr (PH == PH_GU) {
              const float up = __shfl_down_sync(0xffffffffu, v, 16);
              if (lane < 16) p.act[b * 16 + lane] = __float2bfloat16_rn(v / (1.f + __expf(-v)) * up);
            } else {
              const int r = b * kTR + lane;
              if (r < p.vocab_text) best.push(v, r);
            }
          }
          ++blk;
          acc[0] = acc[1] = acc[2] = acc[3] = 0.f;
        }
        if (++k == kt) {
          k = 0;
          ++b;
        }
      }
    }
  }
  // LM head: warp 0's lanes each tracked their own rows; lane 0 reports the merge
  if constexpr (PH == PH_LM) {
    if (warp == 0) warp_top2(best);
  }
}

SR_DEV float mk_qkv_val(const MkParams& p, const __nv_bfloat16* bias, const uint16_t* tab,
                        int row) {
  return mk_sum_parts(p.part_qkv, tab, row, p.maxj) + bf_to_f(bias[row]);
}

// K and V pages land in shared memory as two 64-position x 64-dim boxes each
// (dims 0-63, 64-127; 8 KB), 128-B swizzled by TMA: 16-B chunk c of position
// r sits at r * 128 + ((c ^ (r & 7)) << 4), so the 8 rows of every 8x8
// ldmatrix block fall on distinct banks.  Two TMA ops per page (the pools'
// tensor maps follow the weight maps in p.maps).
constexpr int kQRow = kHeadDim + 8;                  // staged q rows (8 heads), padded
constexpr int kPRow = kPage + 8;                     // staged P rows (bf16), padded
constexpr int kKvTile = kPage * 64 * 2;              // one 64 x 64 box

SR_DEV uint32_t kv_swz(int r, int chunk) {  // byte offset of (position r, 16-B chunk 0..15)
  return (chunk >> 3) * kKvTile + r * 128 + (((chunk & 7) ^ (r & 7)) << 4);
}

// thread 0: one page of the K (which = 0) or V (1) pool (kv head g of `layer`) -> dst
SR_DEV void mk_fetch_tile(const MkParams& p, int which, int layer, int g, int page, uint8_t* dst,
                          uint64_t* bar) {
  const CUtensorMap* map = p.maps + p.L * 4 + 1 + which;
  const int row = (int)((((size_t)layer * p.n_pages + page) * p.KV + g) * kPage);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, 2 * kKvTile);
  tma_load_2d(dst, map, bar, 0, row);
  tma_load_2d(dst + kKvTile, map, bar, 64, row);
}

SR_DEV void ldsm_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(addr));
}
SR_DEV void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
SR_DEV void ldsm_x4t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// m16n8k16 bf16 MMA, fp32 accumulate; rows 8-15 of A are zero (<= 8 heads)
SR_DEV void mma16816(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

SR_DEV void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
SR_DEV void bar_arrive_n(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Pipelined page loop (two page buffers): warps 0-7 (the S group) run S and
// the softmax of page k while warps 8-15 (the V group) run P.V of page k - 1.
//   S group, page k: wait K(k) | S | row max over the group (bar 2) | fetch
//     K(k+2) into the freed buffer | P(k) hi/lo + alpha(k) into P buffer k&1
//     (after the V group released it: bar 5 + (k&1)) | arrive bar 3 + (k&1)
//   V group, page k: sync bar 3 + (k&1) | wait V(k) | O *= alpha(k) | P.V
//     (warp 8 + v: dims 16v..16v+15) | bar 7 | fetch V(k+2) | arrive bar 5 + (k&1)
// Each warp of the S group keeps the l partial of its 8 positions (rescaled
// by alpha like O); they are summed once at the end.
SR_DEV void mk_attn_pipelined(const MkParams& p, int layer, int g, int pos, const int* page_table,
                              int p0, int np, bool has_new, int nh, int jl, int c,
                              uint8_t* const* kvb, uint64_t* kvbar, uint32_t& kvpar,
                              uint32_t q_addr, uint32_t p_addr, uint32_t lo_off, uint32_t pb_stride,
                              __nv_bfloat16* pbh, __nv_bfloat16* pbl, float* red_max, float* red_sum,
                              float* alpha_s, const __nv_bfloat16* knb, const __nv_bfloat16* vnb) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gr = lane >> 2, tq = lane & 3;
  const float scale = 1.4426950408889634f * 0.08838834764831845f;
  auto fetch = [&](int k, int which) {
    const int b = k & 1;
    mk_fetch_tile(p, which, layer, g, page_table[p0 + k], kvb[b] + which * 2 * kKvTile,
                  kvbar + 2 * b + which);
  };
  uint32_t par = kvpar;
  float* a_out = p.apart + ((size_t)c * kMkMaxGq + jl + gr) * 130;
  if (warp < 8) {
    // ------------------------------------------------------------ S group
    const int kr = 8 * warp + (lane & 7);
    float m_run = -INFINITY, l_part = 0.f;
    for (int k = 0; k < np; ++k) {
      const int b = k & 1;
      const int P0 = (p0 + k) * kPage;
      const int nval = min(kPage, pos + 1 - P0);
      const bool last = has_new && k == np - 1;
      uint8_t* kbuf = kvb[b];
      mbar_wait(kvbar + 2 * b, (par >> (2 * b)) & 1u);
      par ^= 1u << (2 * b);
      if (last) {
        if (tid < kHeadDim / 8)
          *reinterpret_cast<uint4*>(kbuf + kv_swz(nval - 1, tid)) = reinterpret_cast<const uint4*>(knb)[tid];
        bar_sync_n(2, 256);
      }
      float sc[4] = {0.f, 0.f, 0.f, 0.f};
      const uint32_t k_smem = smem_u32(kbuf);
#pragma unroll
      for (int kk = 0; kk < kHeadDim / 16; kk += 2) {
        uint32_t a[4], bb[4];
        ldsm_x4(a, q_addr + kk * 32);
        ldsm_x4(bb, k_smem + kv_swz(kr, 2 * kk + (lane >> 3)));
        mma16816(sc, a[0], a[1], bb[0], bb[1]);
        mma16816(sc, a[2], a[3], bb[2], bb[3]);
      }
      const int c0p = 8 * warp + 2 * tq;
      const float s0 = c0p < nval ? sc[0] * scale : -INFINITY;
      const float s1 = c0p + 1 < nval ? sc[1] * scale : -INFINITY;
      float mx = fmaxf(s0, s1);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      float* rm = red_max + b * 64;
      if (tq == 0) rm[warp * 8 + gr] = mx;
      bar_sync_n(2, 256);  // K(k) consumed, row maxima in
      if (tid == 0 && k + 2 < np) fetch(k + 2, 0);
      float pm = rm[gr];
#pragma unroll
      for (int w2 = 1; w2 < 8; ++w2) pm = fmaxf(pm, rm[w2 * 8 + gr]);
      const float m_new = fmaxf(m_run, pm);
      const float alpha = exp2f(m_run - m_new);
      m_run = m_new;
      const float e0 = exp2f(s0 - m_new), e1 = exp2f(s1 - m_new);
      const __nv_bfloat16 h0 = __float2bfloat16_rn(e0), h1 = __float2bfloat16_rn(e1);
      __nv_bfloat162 hi, lo;
      hi.x = h0;
      hi.y = h1;
      lo.x = __float2bfloat16_rn(e0 - __bfloat162float(h0));
      lo.y = __float2bfloat16_rn(e1 - __bfloat162float(h1));
      float rs = e0 + e1;
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      l_part = l_part * alpha + rs;
      if (k >= 2) bar_sync_n(5 + b, 512);  // the V group is done with P buffer b (page k - 2)
      *reinterpret_cast<__nv_bfloat162*>(pbh + b * 8 * kPRow + gr * kPRow + c0p) = hi;
      *reinterpret_cast<__nv_bfloat162*>(pbl + b * 8 * kPRow + gr * kPRow + c0p) = lo;
      if (warp == 0 && tq == 0) alpha_s[b * 8 + gr] = alpha;
      bar_arrive_n(3 + b, 512);  // P(k), alpha(k) ready
    }
    // consume the V group's last releases (one per page in all)
    for (int k = np > 2 ? np : 2; k < np + 2; ++k) bar_sync_n(5 + (k & 1), 512);
    if (tq == 0) red_sum[warp * 8 + gr] = l_part;
    bar_sync_n(2, 256);
    if (warp == 0 && tq == 0 && gr < nh) {
      float l = red_sum[gr];
#pragma unroll
      for (int w2 = 1; w2 < 8; ++w2) l += red_sum[w2 * 8 + gr];
      a_out[128] = m_run;
      a_out[129] = l;
    }
  } else {
    // ------------------------------------------------------------ V group
    const int v = warp - 8;
    const int vr = (lane >> 3) * 8 + (lane & 7);
    float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int k = 0; k < np; ++k) {
      const int b = k & 1;
      const int P0 = (p0 + k) * kPage;
      const int nval = min(kPage, pos + 1 - P0);
      const bool last = has_new && k == np - 1;
      uint8_t* vbuf = kvb[b] + 2 * kKvTile;
      bar_sync_n(3 + b, 512);  // P(k) ready
      mbar_wait(kvbar + 2 * b + 1, (par >> (2 * b + 1)) & 1u);
      par ^= 1u << (2 * b + 1);
      if (last) {  // new v row; rows past the context zeroed
        for (int t = tid - 256; t < (kPage - nval + 1) * 16; t += 256) {
          const int r = nval - 1 + t / 16, q = t % 16;
          *reinterpret_cast<uint4*>(vbuf + kv_swz(r, q)) =
              r == nval - 1 ? reinterpret_cast<const uint4*>(vnb)[q] : make_uint4(0, 0, 0, 0);
        }
        bar_sync_n(7, 256);
      }
      const float alpha = alpha_s[b * 8 + gr];
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        o[n][0] *= alpha;
        o[n][1] *= alpha;
      }
      const uint32_t v_smem = smem_u32(vbuf), pa = p_addr + b * pb_stride;
#pragma unroll
      for (int ks = 0; ks < kPage / 16; ks += 2) {
        uint32_t ah[4], al[4];
        ldsm_x4(ah, pa + ks * 32);
        ldsm_x4(al, pa + lo_off + ks * 32);
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          uint32_t bb[4];
          ldsm_x4t(bb, v_smem + kv_swz(vr + 16 * ks, 2 * v + n));
          mma16816(o[n], ah[0], ah[1], bb[0], bb[1]);
          mma16816(o[n], al[0], al[1], bb[0], bb[1]);
          mma16816(o[n], ah[2], ah[3], bb[2], bb[3]);
          mma16816(o[n], al[2], al[3], bb[2], bb[3]);
        }
      }
      bar_sync_n(7, 256);  // V(k) and P(k) consumed by the group
      if (tid == 256 && k + 2 < np) fetch(k + 2, 1);
      bar_arrive_n(5 + b, 512);  // P buffer b free
    }
    if (gr < nh) {
#pragma unroll
      for (int n = 0; n < 2; ++n)
        *reinterpret_cast<float2*>(a_out + 16 * v + 8 * n + 2 * tq) = make_float2(o[n][0], o[n][1]);
    }
  }
  // both groups leave with the same barrier phases: buffer b was used by the
  // pages k = b, b + 2, ...; each use flipped its K and V barrier once
  const int n0 = (np + 1) / 2, n1 = np / 2;
  kvpar ^= ((n0 & 1) ? 3u : 0u) | ((n1 & 1) ? 12u : 0u);
  cbar();
}

// Attention of kv head g over pages [p0, p1) for its query heads [jl, jh)
// (<= 8: the MMA's rows 0-7, rows 8-15 zero), on the tensor cores:
//   S = Q.K^T  warps 0-7, warp w = positions 8w..8w+7 of the page (m16n8k16,
//              Q and K by ldmatrix from the padded smem rows)
//   softmax    online, exp2, fp32; P kept as bf16 hi + lo (~16 mantissa bits,
//              the oracle's P is fp32)
//   O += P.V   all 16 warps, warp w = dims 8w..8w+7 (V by ldmatrix.trans)
// K and V have their own mbarriers, so the next page's K is in flight while
// this page's softmax and P.V run.  The new position's k / v (summed from the
// qkv partials here) are written into the staged page rows before use, and V
// rows past the context are zeroed (P is 0 there, but 0 * NaN is not).
// Split partials (m, l, O) go to apart; COMBINE merges them.
SR_DEV void mk_attention(const MkParams& p, int layer, int pos, const int* page_table,
                         const __nv_bfloat16* bias, const uint16_t* tab, int c, int S_a,
                         int hs, int npages, float* sm, uint8_t* kvbuf, uint64_t* kvbar, uint32_t& kvpar) {
  const int Gq = p.H / p.KV;
  const int g = c / S_a, s = (c % S_a) / hs, hp = (c % S_a) % hs, PS = S_a / hs;
  if (g >= p.KV) return;  // uniform per CTA
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gr = lane >> 2, tq = lane & 3;  // MMA fragment row / column pair
  const int p0 = (int)((long long)npages * s / PS), p1 = (int)((long long)npages * (s + 1) / PS);
  const int jl = Gq * hp / hs, jh = Gq * (hp + 1) / hs, nh = jh - jl;
  __nv_bfloat16* qb = reinterpret_cast<__nv_bfloat16*>(sm);          // [8][kQRow]
  __nv_bfloat16* pbh = qb + 8 * kQRow;                               // [2][8][kPRow] P hi
  __nv_bfloat16* pbl = pbh + 2 * 8 * kPRow;                          // [2][8][kPRow] P lo
  float* red_max = reinterpret_cast<float*>(pbl + 2 * 8 * kPRow);    // [2][8 warps][8 rows]
  float* red_sum = red_max + 2 * 64;                                 // [8 warps][8 rows]
  float* alpha_s = red_sum + 64;                                     // [2][8 rows]
  __nv_bfloat16* knb = reinterpret_cast<__nv_bfloat16*>(alpha_s + 16);  // [128] new k
  __nv_bfloat16* vnb = knb + kHeadDim;                                  // [128] new v
  // page buffer b: K at kvb[b], V at kvb[b] + 2 boxes; mbarriers kvbar[2b] (K),
  // kvbar[2b + 1] (V), phase parity in bit j of kvpar for barrier j.  With
  // kv_dbl pages alternate between the two buffers and page k + 2 is fetched
  // as soon as page k is done; else K / V of page k + 1 go out as soon as this
  // page's S / P.V no longer need the single buffer.
  const bool dbl = p.kv_dbl != 0;
  uint8_t* const kvb[2] = {kvbuf, kvbuf + kKvBufBytes};
  const int np = p1 - p0;
  auto fetch = [&](int k, int which) {  // thread 0: K (0) or V (1) of local page k
    const int b = dbl ? (k & 1) : 0;
    mk_fetch_tile(p, which, layer, g, page_table[p0 + k], kvb[b] + which * 2 * kKvTile,
                  kvbar + 2 * b + which);
  };
  const float scale = 1.4426950408889634f * 0.08838834764831845f;  // log2(e) / sqrt(128)

  const bool sub_prof = p.prof && c == 0 && tid == 0 && layer == 1;
  int sev = 0;
#define SUB_EV() \
  do { if (sub_prof && sev < 32) p.prof[1600 + sev++] = global_ns(); } while (0)
  SUB_EV();
  // first page's K / V copies go out before anything else (independent of q)
  if (tid == 0) {
    fetch(0, 0);
    fetch(0, 1);
    if (dbl && np > 1) {
      fetch(1, 0);
      fetch(1, 1);
    }
  }
  // q of this CTA's heads: qkv partials + bias, RoPE, bf16 (the oracle's
  // storage point); rows nh..7 zero
  for (int t = tid; t < 8 * kHalf; t += kMkConsumers) {
    const int r = t / kHalf, i = t % kHalf;
    float y0 = 0.f, y1 = 0.f;
    if (r < nh) {
      const int r0 = (g * Gq + jl + r) * kHeadDim + i;
      const float v0 = mk_qkv_val(p, bias, tab, r0), v1 = mk_qkv_val(p, bias, tab, r0 + kHalf);
      const float cs = p.rope[((size_t)pos * kHalf + i) * 2], sn = p.rope[((size_t)pos * kHalf + i) * 2 + 1];
      y0 = v0 * cs - v1 * sn;
      y1 = v1 * cs + v0 * sn;
    }
    qb[r * kQRow + i] = __float2bfloat16_rn(y0);
    qb[r * kQRow + i + kHalf] = __float2bfloat16_rn(y1);
  }
  const bool has_new = p1 == npages;
  if (has_new) {  // new position: k / v from the partials; appended to the pool
    const int page = page_table[pos / kPage];
    const size_t base = kv_offset(layer, page, g, pos % kPage, p.n_pages, p.KV);
    if (tid < kHalf) {
      const int r0 = p.q_dim + g * kHeadDim + tid;
      const float v0 = mk_qkv_val(p, bias, tab, r0), v1 = mk_qkv_val(p, bias, tab, r0 + kHalf);
      const float cs = p.rope[((size_t)pos * kHalf + tid) * 2];
      const float sn = p.rope[((size_t)pos * kHalf + tid) * 2 + 1];
      const __nv_bfloat16 y0 = __float2bfloat16_rn(v0 * cs - v1 * sn);
      const __nv_bfloat16 y1 = __float2bfloat16_rn(v1 * cs + v0 * sn);
      if (hp == 0) {  // one head part appends the new position
        p.k_pool[base + tid] = y0;
        p.k_pool[base + tid + kHalf] = y1;
      }
      knb[tid] = y0;
      knb[tid + kHalf] = y1;
    } else if (tid < kHalf + kHeadDim) {
      const int d2 = tid - kHalf;
      const int r = p.q_dim + p.kv_dim + g * kHeadDim + d2;
      const __nv_bfloat16 y = __float2bfloat16_rn(mk_qkv_val(p, bias, tab, r));
      if (hp == 0) p.v_pool[base + d2] = y;
      vnb[d2] = y;
    }
  }
  float o[4] = {0.f, 0.f, 0.f, 0.f};  // O rows gr (c0, c1) of dims 8*warp + 2*tq, +1
  float m_run = -INFINITY, l_run = 0.f;  // row gr, identical in every thread of the row
  cbar();
  SUB_EV();  // q / new k,v ready
  const uint32_t q_addr = smem_u32(qb) + (lane & 7) * kQRow * 2 + (lane >> 3) * 16;
  // K: position 8w + (lane & 7), chunk 2kk + (lane >> 3); V: position
  // (lane >> 3) * 8 + (lane & 7) (+16ks), chunk w (dims 8w..8w+7)
  const int kr = 8 * (warp & 7) + (lane & 7), vr = (lane >> 3) * 8 + (lane & 7);
  const uint32_t p_addr = smem_u32(pbh) + (lane & 7) * kPRow * 2 + (lane >> 3) * 16;
  const uint32_t lo_off = (uint32_t)(pbl - pbh) * 2, pb_stride = 8 * kPRow * 2;
  if (dbl) {
    mk_attn_pipelined(p, layer, g, pos, page_table, p0, np, has_new, nh, jl, c, kvb, kvbar, kvpar,
                      q_addr, p_addr, lo_off, pb_stride, pbh, pbl, red_max, red_sum, alpha_s, knb, vnb);
    SUB_EV();
    return;
  }

  for (int k = 0; k < np; ++k) {
    const int pg_i = p0 + k;
    const int P0 = pg_i * kPage;
    const int nval = min(kPage, pos + 1 - P0);
    const bool last = has_new && pg_i == p1 - 1;  // holds the new position at nval - 1
    const int b = dbl ? (k & 1) : 0;
    uint8_t* kbuf = kvb[b];
    uint8_t* vbuf = kbuf + 2 * kKvTile;
    const uint32_t k_smem = smem_u32(kbuf), v_smem = smem_u32(vbuf);
    mbar_wait(kvbar + 2 * b, (kvpar >> (2 * b)) & 1u);
    kvpar ^= 1u << (2 * b);
    if (last) {
      if (tid < kHeadDim / 8)
        *reinterpret_cast<uint4*>(kbuf + kv_swz(nval - 1, tid)) = reinterpret_cast<const uint4*>(knb)[tid];
      cbar();
    }
    SUB_EV();  // page landed
    if (warp < 8) {  // S for positions 8w..8w+7, rows gr: c0, c1 = positions 8w + 2tq, +1
      float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < kHeadDim / 16; kk += 2) {
        uint32_t a[4], b[4];
        ldsm_x4(a, q_addr + kk * 32);   // rows 0-7: dims 16kk..+7, +8..15, 16(kk+1).., +8..
        ldsm_x4(b, k_smem + kv_swz(kr, 2 * kk + (lane >> 3)));  // positions 8w..+7: same dims
        mma16816(sc, a[0], a[1], b[0], b[1]);
        mma16816(sc, a[2], a[3], b[2], b[3]);
      }
      const int c0p = 8 * warp + 2 * tq;
      const float s0 = c0p < nval ? sc[0] * scale : -INFINITY;
      const float s1 = c0p + 1 < nval ? sc[1] * scale : -INFINITY;
      float mx = fmaxf(s0, s1);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      if (tq == 0) red_max[warp * 8 + gr] = mx;
      sc[0] = s0;
      sc[1] = s1;
      cbar();  // (1) page max partials in; K buffer free
      if (tid == 0 && !dbl && k + 1 < np) fetch(k + 1, 0);
      float pm = red_max[gr];
#pragma unroll
      for (int w2 = 1; w2 < 8; ++w2) pm = fmaxf(pm, red_max[w2 * 8 + gr]);
      const float m_new = fmaxf(m_run, pm);
      const float e0 = exp2f(s0 - m_new), e1 = exp2f(s1 - m_new);
      const __nv_bfloat16 h0 = __float2bfloat16_rn(e0), h1 = __float2bfloat16_rn(e1);
      __nv_bfloat162 hi, lo;
      hi.x = h0;
      hi.y = h1;
      lo.x = __float2bfloat16_rn(e0 - __bfloat162float(h0));
      lo.y = __float2bfloat16_rn(e1 - __bfloat162float(h1));
      *reinterpret_cast<__nv_bfloat162*>(pbh + gr * kPRow + c0p) = hi;
      *reinterpret_cast<__nv_bfloat162*>(pbl + gr * kPRow + c0p) = lo;
      float rs = e0 + e1;
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      if (tq == 0) red_sum[warp * 8 + gr] = rs;
    } else {
      cbar();  // (1)
    }
    // every thread: the rows' new max and the rescale of its O / l
    float pm = red_max[gr];
#pragma unroll
    for (int w2 = 1; w2 < 8; ++w2) pm = fmaxf(pm, red_max[w2 * 8 + gr]);
    const float m_new = fmaxf(m_run, pm);
    const float alpha = exp2f(m_run - m_new);
    m_run = m_new;
    o[0] *= alpha;
    o[1] *= alpha;
    mbar_wait(kvbar + 2 * b + 1, (kvpar >> (2 * b + 1)) & 1u);
    kvpar ^= 1u << (2 * b + 1);
    if (last) {  // new v row; rows past the context zeroed
      for (int t = tid; t < (kPage - nval + 1) * 16; t += kMkConsumers) {
        const int r = nval - 1 + t / 16, q = t % 16;
        *reinterpret_cast<uint4*>(vbuf + kv_swz(r, q)) =
            r == nval - 1 ? reinterpret_cast<const uint4*>(vnb)[q] : make_uint4(0, 0, 0, 0);
      }
    }
    cbar();  // (2) P, row sums and the staged V in
    {
      float rs = red_sum[gr];
#pragma unroll
      for (int w2 = 1; w2 < 8; ++w2) rs += red_sum[w2 * 8 + gr];
      l_run = l_run * alpha + rs;
    }
#pragma unroll
    for (int ks = 0; ks < kPage / 16; ks += 2) {
      uint32_t ah[4], al[4], b[4];
      ldsm_x4(ah, p_addr + ks * 32);
      ldsm_x4(al, p_addr + lo_off + ks * 32);
      ldsm_x4t(b, v_smem + kv_swz(vr + 16 * ks, warp));  // positions 16ks..16ks+31, dims 8w..+7
      mma16816(o, ah[0], ah[1], b[0], b[1]);
      mma16816(o, al[0], al[1], b[0], b[1]);
      mma16816(o, ah[2], ah[3], b[2], b[3]);
      mma16816(o, al[2], al[3], b[2], b[3]);
    }
    cbar();  // (3) V, P and the row partials free
    if (tid == 0) {
      if (!dbl && k + 1 < np) fetch(k + 1, 1);
      if (dbl && k + 2 < np) {
        fetch(k + 2, 0);
        fetch(k + 2, 1);
      }
    }
    SUB_EV();
  }
  // partials: O rows gr < nh (head jl + gr), dims 8w + 2tq, +1; m / l
  if (gr < nh) {
    float* a = p.apart + ((size_t)c * kMkMaxGq + jl + gr) * 130;
    *reinterpret_cast<float2*>(a + 8 * warp + 2 * tq) = make_float2(o[0], o[1]);
    if (warp == 0 && tq == 0) {
      a[128] = m_run;
      a[129] = l_run;
    }
  }
  SUB_EV();  // partial written
#undef SUB_EV
}

// COMBINE: merge the attention splits.  Work item = (query head, 32·NW-dim
// slice), spread over the grid; 16 thread groups each take every 16th split,
// one round trip of loads, then a fixed-order merge of the groups
// (deterministic).  NW = 2 (64-dim items, float2 loads) when 32-dim items
// would outnumber the CTAs (32B: 160 items on 148 CTAs, so 12 CTAs ran two
// rounds and every CTA waited for them at the next barrier); the arithmetic
// per (head, dim) is the same sequence either way, so the result is
// bit-identical.  The width is a kernel template parameter (mk_launch).
template <int NW>
SR_DEV void mk_combine_w(const MkParams& p, int c, int G, int S_a, int hs, float* sm) {
  constexpr int W = 32 * NW, PER = kHeadDim / W, B = 4 / NW;  // B splits in flight
  const int Gq = p.H / p.KV;
  const int tid = threadIdx.x, dl = tid & 31, grp = tid >> 5;
  float* r_o = sm;                  // [16][W]
  float* r_m = sm + kMkWarps * W;   // [16]
  float* r_l = r_m + kMkWarps;      // [16]
  for (int it = c; it < p.H * PER; it += G) {
    const int h = it / PER, d = (it % PER) * W + dl * NW;
    const int g = h / Gq, j = h - g * Gq;
    // with head splits only the part owning head j holds data: splits s*hs + hp
    int hp = 0;
    while (hp + 1 < hs && Gq * (hp + 1) / hs <= j) ++hp;
    float m = -INFINITY, l = 0.f, o[NW];
#pragma unroll
    for (int e = 0; e < NW; ++e) o[e] = 0.f;
    // this group's splits q0, q0 + qs, ...: B at a time, all loads issued
    // before the (in-order, so unchanged) merge -- one L2 round trip per B
    const int q0 = grp * hs + hp, qs = kMkWarps * hs;
    for (int qb = q0; qb < S_a; qb += B * qs) {
      float ms[B], ls[B], os[B][NW];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const int q = qb + i * qs;
        ms[i] = -INFINITY;
        ls[i] = 0.f;
#pragma unroll
        for (int e = 0; e < NW; ++e) os[i][e] = 0.f;
        if (q < S_a) {
          const float* a = p.apart + ((size_t)(g * S_a + q) * kMkMaxGq + j) * 130;
          ms[i] = __ldcg(a + 128);
          ls[i] = __ldcg(a + 129);
          if constexpr (NW == 2) {
            const float2 v = __ldcg(reinterpret_cast<const float2*>(a + d));  // 130·4 B rows: 8-B aligned
            os[i][0] = v.x;
            os[i][1] = v.y;
          } else {
            os[i][0] = __ldcg(a + d);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < B; ++i) {
        if (ms[i] == -INFINITY) continue;  // past S_a, or a head-split slot of another head
        const float mn = fmaxf(m, ms[i]);
        const float x = exp2f(m - mn), y = exp2f(ms[i] - mn);
        l = l * x + ls[i] * y;
#pragma unroll
        for (int e = 0; e < NW; ++e) o[e] = o[e] * x + os[i][e] * y;
        m = mn;
      }
    }
#pragma unroll
    for (int e = 0; e < NW; ++e) r_o[grp * W + dl * NW + e] = o[e];
    if (dl == 0) {
      r_m[grp] = m;
      r_l[grp] = l;
    }
    cbar();
    if (grp == 0) {
      float M = r_m[0], L = r_l[0], O[NW];
#pragma unroll
      for (int e = 0; e < NW; ++e) O[e] = r_o[dl * NW + e];
      for (int q = 1; q < kMkWarps; ++q) {
        const float mq = r_m[q];
        if (mq == -INFINITY) continue;
        const float mn = fmaxf(M, mq);
        const float x = exp2f(M - mn), y = exp2f(mq - mn);
        L = L * x + r_l[q] * y;
#pragma unroll
        for (int e = 0; e < NW; ++e) O[e] = O[e] * x + r_o[q * W + dl * NW + e] * y;
        M = mn;
      }
#pragma unroll
      for (int e = 0; e < NW; ++e) p.attn[(size_t)h * kHeadDim + d + e] = __float2bfloat16_rn(O[e] / L);
    }
    cbar();
  }
}

// Walks this CTA's tile sequence: per token, layer 0..L-1 x (qkv, o, gate/up,
// down), then the LM head; wraps to the next token.  Empty phases are skipped.
struct MkCursor {
  int l, k, u, hi, kk, bb, kt, tc, bytes;
  const CUtensorMap* map;
  const uint8_t* tbase;  // tile-major weights of the phase (p.tiled)
  SR_DEV void enter(const MkParams& p, const PhaseInfo* ph) {
    for (;;) {
      const PhaseInfo& pi = ph[l < p.L ? k : PH_LM];
      map = p.maps + (l < p.L ? l * 4 + k : p.L * 4);
      tbase = p.tiled ? static_cast<const uint8_t*>(p.tiles[l < p.L ? l * 4 + k : p.L * 4]) : nullptr;
      u = pi.lo;
      hi = pi.hi;
      kk = pi.k0;
      bb = pi.b0;
      kt = pi.kt;
      tc = pi.tc;
      bytes = pi.bytes;
      if (u < hi) return;
      step_phase(p);
    }
  }
  SR_DEV void step_phase(const MkParams& p) {
    if (l < p.L && ++k < 4) return;
    k = 0;
    if (++l > p.L) l = 0;
  }
  SR_DEV void init(const MkParams& p, const PhaseInfo* ph) {
    l = 0;
    k = 0;
    enter(p, ph);
  }
  SR_DEV void next(const MkParams& p, const PhaseInfo* ph) {
    if (++kk == kt) {
      kk = 0;
      ++bb;
    }
    if (++u < hi) return;
    step_phase(p);
    enter(p, ph);
  }
  SR_DEV int col() const { return kk * tc; }
  SR_DEV int row() const { return bb * kTR; }
  SR_DEV const uint8_t* tile() const { return tbase + ((size_t)bb * kt + kk) * bytes; }
};

SR_DEV void l2_prefetch(const void* ptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// Layer l's small vectors (norm weights, qkv bias) and this CTA's attention
// pages, pulled into L2 a layer early: under the weight stream an HBM miss
// costs several microseconds on the latency-bound path (l == L: next token).
SR_DEV void mk_prefetch_next_layer(const MkParams& p, int l, int pos, const int* page_table,
                                   int c, int G, int S_a, int hs, int npages) {
  if (l >= p.L) {  // layer 0 of the next token: its RoPE row too
    l = 0;
    ++pos;
  }
  if (c == 1) l2_prefetch(p.rope + (size_t)pos * kHalf * 2, kHalf * 2 * 4);
  if (c == 0) {
    const MkLayer ly = p.layers[l];
    l2_prefetch(ly.ln1, p.d * 2);
    l2_prefetch(ly.ln2, p.d * 2);
    l2_prefetch(ly.bqkv, p.qkv_rows * 2);
  }
  const int g = c / S_a, s = (c % S_a) / hs, PS = S_a / hs;
  if (g >= p.KV || (c % S_a) % hs != 0) return;  // one head part prefetches the pages
  const int p0 = (int)((long long)npages * s / PS), p1 = (int)((long long)npages * (s + 1) / PS);
  for (int pg = p0; pg < p1; ++pg) {
    const size_t off = kv_offset(l, page_table[pg], g, 0, p.n_pages, p.KV);
    l2_prefetch(p.k_pool + off, kPage * kHeadDim * 2);
    l2_prefetch(p.v_pool + off, kPage * kHeadDim * 2);
  }
}

// kTiled: the tile-major weights + mma.sync consumers (p.tiled), else row-major
// TMA boxes + CUDA-core consumers; two instantiations, so each carries the
// registers of one consumer only
template <bool kTiled, bool kWide>
__global__ void __launch_bounds__(kMkThreads, 1) decode_mk_kernel(const MkParams p) {
  extern __shared__ __align__(1024) uint8_t mk_smem[];
  __shared__ __align__(8) uint64_t full[kMkMaxStages];
  __shared__ __align__(8) uint64_t empty[kMkMaxStages];
  __shared__ float red[32];
  __shared__ float s_v1[kMkWarps], s_v2[kMkWarps];
  __shared__ int s_i1[kMkWarps];
  __shared__ int s_tok;
  __shared__ uint16_t s_tab[3][kMkTab];  // contributor tables: qkv, o, down
  __shared__ float s_gred[2 * 256];       // mma GEMV: per-row-block slice sums, 2 buffers
  __shared__ PhaseInfo s_ph[5];
  __shared__ __align__(8) uint64_t kvbar[4];  // K, V of page buffer 0; K, V of buffer 1
  __shared__ float s_margin, s_rv1, s_rv2;
  __shared__ volatile int s_stop;

  const int S = p.stages;
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = mk_smem;
  uint8_t* kvbuf = mk_smem + (size_t)S * kStageBytes;  // one K page + one V page
  float* kvtmp = reinterpret_cast<float*>(kvbuf);         // prologue scratch (d <= 5120)
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(kvbuf + kKvBufBytes);
  // attention: second page buffer at xs (1024-aligned), scratch behind it
  float* scratch = reinterpret_cast<float*>(kvbuf + kKvBufBytes + (p.kv_dbl ? kKvBufBytes : 0));

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kMkWarps);
    }
    s_stop = 0;
    for (int i = 0; i < 4; ++i) mbar_init(&kvbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 5) s_ph[threadIdx.x] = mk_phase_info(p, threadIdx.x, blockIdx.x, gridDim.x);
  __syncthreads();

  DecodeState* st = p.st;
  const int L = p.L;

  if (warp == kMkWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      // a CTA with no tiles in any phase (tiny models) has nothing to stream
      int mine = 0;
      for (int ph = 0; ph <= PH_LM; ++ph) mine += s_ph[ph].hi - s_ph[ph].lo;
      uint32_t n = 0;
      if (mine > 0) {
        MkCursor ld, pf;
        ld.init(p, s_ph);
        pf.init(p, s_ph);
        uint32_t npf = 0, nld = 0;  // units prefetched into L2 / loaded
        const uint32_t ahead = (uint32_t)(S * kUPS + (p.l2_ahead > 0 ? p.l2_ahead : 0));
        int slot = 0;
        uint32_t par = 1u;
        const uint64_t pol = l2_policy_evict_first();
        for (;;) {
          // L2 prefetch run-ahead: HBM keeps streaming while the consumers sit
          // in latency-bound phases longer than the shared-memory ring covers
          if (p.l2_ahead >= 0) {
            while (npf < nld + ahead) {
              if (kTiled)  // one contiguous tile of the decode-layout weights
                l2_prefetch(pf.tile(), (uint32_t)pf.bytes);
              else
                tma_prefetch_2d(pf.map, pf.col(), pf.row());
              pf.next(p, s_ph);
              ++npf;
            }
          }
          bool stop = false;
          while (!mbar_try(&empty[slot], par)) {
            if (s_stop) {
              stop = true;
              break;
            }
          }
          if (stop || s_stop) break;
          if (p.trace) p.trace[c * 8 + 3] = (int)n;
          if (p.no_load) {  // experiment: consumer chain without the weight stream
            const int nu = ld.hi - ld.u < kUPS ? ld.hi - ld.u : kUPS;
            for (int q = 0; q < nu; ++q) ld.next(p, s_ph);
            nld += nu;
            mbar_arrive(&full[slot]);
          } else {
            const int nu = ld.hi - ld.u < kUPS ? ld.hi - ld.u : kUPS;
            mbar_expect_tx(&full[slot], nu * ld.bytes);
            uint8_t* dst = ring + (size_t)slot * kStageBytes;
            for (int q = 0; q < nu; ++q) {
              if (kTiled)  // one contiguous 16 KB tile, already in the smem image
                bulk_load_1d_hint(dst + q * kTileBytes, ld.tile(), ld.bytes, &full[slot], pol);
              else if (p.evict_first)
                tma_load_2d_hint(dst + q * kTileBytes, ld.map, &full[slot], ld.col(), ld.row(), pol);
              else
                tma_load_2d(dst + q * kTileBytes, ld.map, &full[slot], ld.col(), ld.row());
              ld.next(p, s_ph);
            }
            nld += nu;
          }
          ++n;
          if (++slot == S) {
            slot = 0;
            par ^= 1u;
          }
        }
      }
      // let every issued copy land before the CTA exits
      for (uint32_t m = n > (uint32_t)S ? n - (uint32_t)S : 0u; m < n; ++m)
        mbar_wait(&full[m % (uint32_t)S], (m / (uint32_t)S) & 1u);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  if (p.no_load)  // experiment: the unloaded ring reads as zeros (finite results)
    for (int i = threadIdx.x; i < S * kStageBytes / 16; i += kMkConsumers)
      reinterpret_cast<uint4*>(ring)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < 3 * kMkTab; i += kMkConsumers) (&s_tab[0][0])[i] = p.ctab[i];
  cbar();
  int pos = st->pos, tok = st->token, n_gen = st->n_gen;
  const int max_new = st->max_new;
  const int* page_table = st->page_table;
  const uint8_t* token_class = st->token_class;
  unsigned* bar = &st->bar;
  unsigned target = 0;
  RingPos rp{0, 0u};
  uint32_t kvpar = 0u;
  const int Gq = p.H / p.KV;
  (void)Gq;
  bool done = st->done != 0;
  // tensor parallelism: exchange counters continue across launches (words 8-9
  // of this rank's buffer; every rank runs the same exchange sequence)
  const bool tp = p.tp_world > 1;
  unsigned* tp_ctr = tp ? reinterpret_cast<unsigned*>(p.tp_base[p.tp_rank]) + 8 : nullptr;
  unsigned ex = tp ? tp_ctr[0] : 0u, lx = tp ? tp_ctr[1] : 0u;
  const float* mb_d = nullptr;  // mailbox slot of the last down exchange
  // SR_MK_PROF: CTA 0 records a globaltimer stamp after every step of the
  // first decoded token (sr_debug_profile)
  const bool prof = p.prof != nullptr && c == 0 && threadIdx.x == 0;
  int ev = 0;
  int tstep = 0;
#define MK_EV()                                                                        \
  do {                                                                                 \
    if (prof && ev < kMkProfEvents) p.prof[ev++] = global_ns();                        \
    if (p.trace && threadIdx.x == 0) {                                                 \
      volatile int* tr = p.trace + c * 8;                                              \
      tr[0] = ++tstep;                                                                 \
      tr[1] = rp.slot;                                                                 \
      tr[2] = (int)target;                                                             \
      tr[4] = n_gen;                                                                   \
    }                                                                                  \
  } while (0)

  while (!done) {
    MK_EV();
    const int npages = pos / kPage + 1;
    // splits per kv head: the fewest that keep the largest split at the page
    // count the CTAs allow (96 pages over 74 CTAs would hold 1 or 2 pages
    // each; 48 splits of 2 pages finish at the same time with less COMBINE
    // work: 1.5B at 6 K 1.153 -> 1.123 ms/token)
    const int smax = G / p.KV;
    int per = (npages + smax - 1) / smax;
    if (per < p.min_pages) per = p.min_pages;
    int S_a = (npages + per - 1) / per;
    if (S_a > smax) S_a = smax;
    if (S_a < 1) S_a = 1;
    // more CTAs than page splits (short contexts): split each page's query
    // heads over hs CTAs too, so idle CTAs share the per-page latency chain
    int hs = p.head_split ? (G / p.KV) / S_a : 1;
    if (hs > p.H / p.KV) hs = p.H / p.KV;
    if (hs < 1) hs = 1;
    S_a *= hs;
    Top2 best;
    best.init();
    for (int l = 0; l < L; ++l) {
      const MkLayer ly = p.layers[l];
      // QKV
      if (l == 0)
        mk_norm_prologue(p, 0, tok, nullptr, nullptr, s_tab[2], ly.ln1, p.hA, xs, red, c, G, kvtmp);
      else
        mk_norm_prologue(p, 1, tok, p.hB, p.part_d, s_tab[2], ly.ln1, p.hA, xs, red, c, G, kvtmp,
                         mb_d, l == 1 && tstep < 40 ? 1640 : -1);
      MK_EV();  // 1 qkv prologue
      if constexpr (kTiled) mk_gemv_mma<PH_QKV>(p, s_ph[PH_QKV], c, ring, full, empty, xs, rp, S, best, s_gred); else mk_gemv<PH_QKV>(p, s_ph[PH_QKV], c, ring, full, empty, xs, rp, S, best);
      MK_EV();  // 2 qkv gemv
      mk_grid_sync(bar, target, G, p.bar_sleep);
      MK_EV();  // 3 sync
      // attention (+ merge of the splits by the last split CTA of each kv head)
      const uint64_t ta0 = global_ns();
      mk_attention(p, l, pos, page_table, ly.bqkv, s_tab[0], c, S_a, hs, npages, scratch, kvbuf,
                   kvbar, kvpar);
      if (p.prof && threadIdx.x == 0 && l == 1 && tstep < 40) {  // per-CTA attention time, layer 1
        p.prof[1280 + c] = global_ns() - ta0;
        p.prof[1440 + c] = (c % S_a) == S_a - 1;
      }
      // warm L2 with what the next layer reads on its latency-bound path
      if (threadIdx.x == 0)
        mk_prefetch_next_layer(p, l + 1, pos, page_table, c, G, S_a, hs, npages);
      MK_EV();  // 4 attention
      mk_grid_sync(bar, target, G, p.bar_sleep);
      MK_EV();  // 5 sync
      if constexpr (kWide) mk_combine_w<2>(p, c, G, S_a, hs, scratch); else mk_combine_w<1>(p, c, G, S_a, hs, scratch);
      MK_EV();  // 6 combine
      mk_grid_sync(bar, target, G, p.bar_sleep);
      MK_EV();  // 7 sync
      // O
      mk_stage_vec(p.attn, p.q_dim, xs);
      MK_EV();  // 8 stage
      if constexpr (kTiled) mk_gemv_mma<PH_O>(p, s_ph[PH_O], c, ring, full, empty, xs, rp, S, best, s_gred); else mk_gemv<PH_O>(p, s_ph[PH_O], c, ring, full, empty, xs, rp, S, best);
      MK_EV();  // 9 o gemv
      mk_grid_sync(bar, target, G, p.bar_sleep);
      MK_EV();  // 10 sync
      const float* mb_o = tp ? mk_tp_exchange(p, p.part_o, s_tab[1], ex, c, G) : nullptr;
      // gate / up
      mk_norm_prologue(p, 1, tok, p.hA, p.part_o, s_tab[1], ly.ln2, p.hB, xs, red, c, G, kvtmp,
                       mb_o, l == 1 && tstep < 40 ? 1650 : -1);
      MK_EV();  // 11 prologue
      if constexpr (kTiled) mk_gemv_mma<PH_GU>(p, s_ph[PH_GU], c, ring, full, empty, xs, rp, S, best, s_gred); else mk_gemv<PH_GU>(p, s_ph[PH_GU], c, ring, full, empty, xs, rp, S, best);
      MK_EV();  // 12 gu gemv
      mk_grid_sync(bar, target, G, p.bar_sleep);
      MK_EV();  // 13 sync
      // down
      mk_stage_vec(p.act, p.f, xs);
      MK_EV();  // 14 stage
      if constexpr (kTiled) mk_gemv_mma<PH_D>(p, s_ph[PH_D], c, ring, full, empty, xs, rp, S, best, s_gred); else mk_gemv<PH_D>(p, s_ph[PH_D], c, ring, full, empty, xs, rp, S, best);
      MK_EV();  // 15 down gemv
      mk_grid_sync(bar, target, G, p.bar_sleep);
      MK_EV();  // 16 sync
      if (tp) mb_d = mk_tp_exchange(p, p.part_d, s_tab[2], ex, c, G);
    }
    // LM head + greedy argmax
    mk_norm_prologue(p, 1, tok, p.hB, p.part_d, s_tab[2], p.ln_f, nullptr, xs, red, c, G, kvtmp,
                     mb_d);
    MK_EV();
    if constexpr (kTiled) mk_gemv_mma<PH_LM>(p, s_ph[PH_LM], c, ring, full, empty, xs, rp, S, best, s_gred); else mk_gemv<PH_LM>(p, s_ph[PH_LM], c, ring, full, empty, xs, rp, S, best);
    MK_EV();
    if (lane == 0) {
      s_v1[warp] = best.v1;
      s_v2[warp] = best.v2;
      s_i1[warp] = best.i1;
    }
    cbar();
    if (threadIdx.x == 0) {
      Top2 b;
      b.init();
      for (int w = 0; w < kMkWarps; ++w) b.merge(s_v1[w], s_i1[w], s_v2[w]);
      p.lm_part[c * 3 + 0] = b.v1;
      p.lm_part[c * 3 + 1] = b.v2;
      p.lm_part[c * 3 + 2] = __int_as_float(b.i1);
    }
    mk_grid_sync(bar, target, G, p.bar_sleep);
    MK_EV();
    if (warp == 0) {
      Top2 b;
      b.init();
      for (int i = lane; i < G; i += 32)
        b.merge(__ldcg(p.lm_part + i * 3), __float_as_int(__ldcg(p.lm_part + i * 3 + 2)),
                __ldcg(p.lm_part + i * 3 + 1));
      warp_top2(b);
      if (lane == 0) {
        s_tok = b.i1;
        s_rv1 = b.v1;
        s_rv2 = b.v2;
        s_margin = b.v1 - b.v2;
      }
    }
    cbar();
    if (tp) {  // this rank's vocab shard -> global greedy choice over all ranks
      Top2 mine;
      mine.v1 = s_rv1;
      mine.v2 = s_rv2;
      mine.i1 = s_tok + p.vocab_base;
      const Top2 b = mk_tp_merge(p, mine, lx, c);
      if (threadIdx.x == 0) {
        s_tok = b.i1;
        s_margin = b.v1 - b.v2;
      }
      cbar();
    }
    const int t = s_tok;
    const int cls = token_class[t];
    int finish = SR_FINISH_LENGTH;
    done = false;
    if (cls == SR_CLASS_END_THINK) {
      done = true;
      finish = SR_FINISH_END_THINK;
    } else if (cls == SR_CLASS_STOP) {
      done = true;
      finish = SR_FINISH_STOP;
    } else if (n_gen + 1 >= max_new) {
      done = true;
    }
    if (c == 0 && threadIdx.x == 0) {
      st->out_ids[n_gen] = t;
      if (st->margins) st->margins[n_gen] = s_margin;
      st->n_gen = n_gen + 1;
      st->done = done ? 1 : 0;
      st->finish = finish;
      if (!done) {
        st->token = t;
        st->pos = pos + 1;
        st->ctx_len = pos + 2;
      }
      st->out_hdr[0] = n_gen + 1;
      st->out_hdr[1] = finish;
    }
    n_gen += 1;
    tok = t;
    pos += 1;
    MK_EV();
    if (prof) ev = kMkProfEvents;  // first token only
  }
#undef MK_EV
  if (tp && c == 0 && threadIdx.x == 0) {
    tp_ctr[0] = ex;
    tp_ctr[1] = lx;
  }
  if (threadIdx.x == 0) s_stop = 1;
}

// ------------------------------------------------------------------- host ---
// ring | K/V page buffer | vector region: the GEMV input x, which during
// attention holds the attention scratch and, with kv_dbl, a second K/V page
// buffer in front of it
size_t mk_smem_bytes(int stages, int xs_elems, int kv_dbl) {
  size_t xs = (size_t)xs_elems * 2;
  const size_t attn = (size_t)kMkAttnScratchFloats * 4 + (kv_dbl ? kKvBufBytes : 0);
  if (xs < attn) xs = attn;
  return (size_t)stages * kStageBytes + kKvBufBytes + xs;
}

int mk_pick_stages(int xs_elems) {
  int s = kMkMaxStages;
  while (s > 2 && mk_smem_bytes(s, xs_elems, 0) > 222 * 1024) --s;  // + <= 5 KB static
  return s;
}

// double-buffer the attention pages when that costs no ring stage
int mk_pick_kv_dbl(int stages, int xs_elems) {
  return mk_smem_bytes(stages, xs_elems, 1) <= 222 * 1024 ? 1 : 0;
}

int mk_max_j(int N, int K, int num_sms) {
  const int kt = (K + kTC - 1) / kTC, nb = (N + kTR - 1) / kTR;
  const int T = nb * kt;
  const int per = (T + num_sms - 1) / num_sms;
  return per > 0 ? (per - 1) / kt + 2 : 1;
}

int mk_tile_rows() { return kTR; }
int mk_tile_cols() { return kTC; }

cudaError_t mk_launch(const MkParams& p, int num_sms, cudaStream_t stream) {
  const size_t smem = mk_smem_bytes(p.stages, p.xs_elems, p.kv_dbl);
  // instantiations: consumer (tile-major mma.sync / row-major CUDA-core) x
  // COMBINE item width, so each carries the registers of its own variants only
  const bool wide = p.combine_wide > 0 || (p.combine_wide < 0 && p.H * (kHeadDim / 32) > num_sms);
  auto* kern = p.tiled ? (wide ? decode_mk_kernel<true, true> : decode_mk_kernel<true, false>)
                       : (wide ? decode_mk_kernel<false, true> : decode_mk_kernel<false, false>);
  static size_t attr[4] = {0, 0, 0, 0};
  size_t& a = attr[(p.tiled ? 2 : 0) + (wide ? 1 : 0)];
  if (a < smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    a = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(kMkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace sr
