// K7 on the 5th-generation tensor cores: paged flash attention for prefill and
// verification (tcgen05.mma, accumulators in TMEM, K/V pages by TMA).
//
// CTA = (kv head g, KV split, 128 query rows); query rows are (token,
// head-in-group) pairs of g, so the G heads sharing a K/V page form the MMA's
// M dimension and every K/V byte is read once per 128-row tile.  4 warps;
// thread t owns query row t, which is TMEM lane t of every accumulator.
//
// Per 64-position page:
//   S = Q K^T      tcgen05.mma M=128 N=64 K=128 (Q and K both K-major, 128-B
//                  swizzled; Q written once by the threads, K by TMA)
//   softmax        tcgen05.ld of the thread's S row, causal mask, exp2 online
//                  softmax in fp32; P split into bf16 hi + lo (the oracle keeps
//                  P in fp32: ~16 mantissa bits survive) and written as the
//                  K-major A operand of the next product
//   O += P V       tcgen05.mma M=128 N=128 K=64 twice (P_hi, P_lo); V is read
//                  straight from its page as an MN-major B operand
// O stays in TMEM for the whole split; when a row's running max moves, the
// warp rescales its 32 rows in place (tcgen05.ld / st).  Splits leave
// (m, l, O) partials for attn_merge_kernel, exactly like attention_tc.cu.
#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace sr {

constexpr int kFaRows = 128;
constexpr int kFaSoftmaxWarps = 8;                  // two threads per query row
constexpr int kFaThreads = kFaSoftmaxWarps * 32 + 32;  // + the TMA / MMA issue warp
constexpr int kFaHalf = 64 * 64 * 2;                 // one [64 x 64] bf16 sub-tile: 8 KB
constexpr int kFaStage = 4 * kFaHalf;                // K (2 halves) + V (2 halves): 32 KB
constexpr int kFaQBytes = 2 * kFaRows * 128;         // Q: 2 x [128 x 64]: 32 KB
constexpr int kFaStages = 2;                         // K/V pages in flight
constexpr int kStageLd = 132;  // fp32 row pitch of the epilogue staging (bank spread)
constexpr int kFaSmem = kFaQBytes + kFaStages * kFaStage + 1024;
static_assert(kFaRows * kStageLd * 4 <= kFaQBytes + kFaStages * kFaStage, "epilogue staging fits");  // 97 KB: 2 CTAs / SM
constexpr float kFaScaleLog2 = 1.4426950408889634f * 0.08838834764831845f;
constexpr float kFaLazy = 8.f;  // log2 headroom of the lazy softmax rescale

// byte offset of (row, 16-B chunk) in a 128-B-swizzled K-major [rows x 64] tile
SR_DEV uint32_t sw128(int row, int chunk) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}

SR_DEV void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

SR_DEV void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

SR_DEV void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}

// 2^x with flush-to-zero: exp2f adds a range fix-up around MUFU.EX2 for
// results below 2^-126 (3 more instructions per score); such probabilities are
// far below the fp32 resolution of the row sums they join
SR_DEV float exp2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

SR_DEV void named_barrier_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// O += P V with P (the A operand) read from tensor memory
SR_DEV void umma_bf16_tmem_a(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__global__ void __launch_bounds__(kFaThreads, 2)
    attn_prefill_umma_kernel(const __grid_constant__ CUtensorMap tmK,
                             const __grid_constant__ CUtensorMap tmV, AttnParams p, int M_rows,
                             int G) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t k_full[kFaStages];
  __shared__ __align__(8) uint64_t v_full[kFaStages];
  __shared__ __align__(8) uint64_t s_full[2];
  __shared__ __align__(8) uint64_t p_full[2];
  __shared__ __align__(8) uint64_t o_done;
  __shared__ uint32_t tmem_s;
  __shared__ float xch[2][2][kFaRows];  // [page parity][half][row]: row max / sum exchange

  const int g = blockIdx.x, split = blockIdx.y;
  // the sequence (span) and query tile of this CTA: one span (rows 0..M_rows)
  // unless p.spans lists (first token, tokens, start position, tile) per z
  int tok0 = 0, span_rows = M_rows, start = p.start_pos, qt = blockIdx.z;
  const int* ptab = p.page_table;
  if (p.spans) {
    const int4 it = p.spans[blockIdx.z];
    tok0 = it.x;
    span_rows = it.y * G;
    start = it.z;
    qt = it.w;
    ptab = p.span_tables[blockIdx.z];
  }
  const int grow0 = tok0 * G;  // first global query row of the span
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool ctrl = warp == kFaSoftmaxWarps;  // TMA + MMA issue warp
  const int r = tid & (kFaRows - 1);          // query row = TMEM lane
  const int hf = (tid >> 7) & 1;              // which 32 of a page's 64 positions / 64 of O's dims
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* base = smem_raw + ((1024 - (raw & 1023)) & 1023);
  uint8_t* sQ = base;
  uint8_t* sKV = sQ + kFaQBytes;

  const int row0 = qt * kFaRows;  // within the span
  const int rows_here = min(kFaRows, span_rows - row0);
  const int last_tok = (row0 + rows_here - 1) / G;
  const int T = start + last_tok + 1;
  const int n_tiles = (T + kPage - 1) / kPage;
  const int nsplit = gridDim.y;
  const int per = (n_tiles + nsplit - 1) / nsplit;
  const int t_lo = split * per;
  const int t_hi = min(n_tiles, t_lo + per);
  const int np = t_hi > t_lo ? t_hi - t_lo : 0;

  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmK) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmV) : "memory");
    for (int i = 0; i < kFaStages; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], kFaSoftmaxWarps * 32);
    }
    mbar_init(&o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     smem_u32(&tmem_s))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  grid_launch_dependents();
  grid_wait();  // q and the new K/V rows come from the predecessor

  // ---- query row r, dims 64*hf .. 64*hf+63 -> Q sub-tile hf (K-major, SW128) ----
  if (!ctrl) {
    uint4 v[8];
    if (r < rows_here) {
      const int rr = row0 + r, tok = tok0 + rr / G, j = rr % G;
      const uint4* src = reinterpret_cast<const uint4*>(
          p.q + (size_t)tok * p.n_heads * kHeadDim + (size_t)(g * G + j) * kHeadDim + 64 * hf);
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = src[c];
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      *reinterpret_cast<uint4*>(sQ + hf * (kFaRows * 128) + sw128(r, c)) = v[c];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_s;
  auto tS = [tmem](int b) { return tmem + 64u * (uint32_t)b; };  // S / P buffers b = 0, 1
  const uint32_t tO = tmem + 128;

  if (ctrl) {
    // ---- control warp, one lane: K/V pages by TMA, S and PV on the tensor core.
    // K of page i lives in stage i % 2 until S_i is done, V until PV_i is.
    if ((tid & 31) == 0 && np > 0) {
      auto page_row = [&](int i) {
        return ((p.layer * p.n_pages + ptab[t_lo + i]) * p.n_kv + g) * kPage;
      };
      auto issue_k = [&](int i) {
        const int st = i % kFaStages;
        uint8_t* d = sKV + st * kFaStage;
        mbar_expect_tx(&k_full[st], 2 * kFaHalf);
        tma_load_2d(d, &tmK, &k_full[st], 0, page_row(i));
        tma_load_2d(d + kFaHalf, &tmK, &k_full[st], 64, page_row(i));
      };
      auto issue_v = [&](int i) {
        const int st = i % kFaStages;
        uint8_t* d = sKV + st * kFaStage + 2 * kFaHalf;
        mbar_expect_tx(&v_full[st], 2 * kFaHalf);
        tma_load_2d(d, &tmV, &v_full[st], 0, page_row(i));
        tma_load_2d(d + kFaHalf, &tmV, &v_full[st], 64, page_row(i));
      };
      const uint32_t idS = umma_idesc(64);
      const uint32_t idO = umma_idesc(128) | (1u << 16);  // B (V) MN-major
      const uint32_t q0 = smem_u32(sQ);
      auto issue_S = [&](int i) {  // S_i = Q K_i^T into tS(i & 1)
        const int st = i % kFaStages;
        mbar_wait(&k_full[st], (uint32_t)(i / kFaStages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t k0 = smem_u32(sKV + st * kFaStage);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (uint32_t)((kk & 3) * 32);
          umma_bf16(tS(i & 1), umma_desc_sw128(q0 + (kk >> 2) * (kFaRows * 128) + off),
                    umma_desc_sw128(k0 + (kk >> 2) * kFaHalf + off), idS, kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[i & 1]);
      };
      for (int i = 0; i < kFaStages && i < np; ++i) {
        issue_k(i);
        issue_v(i);
      }
      issue_S(0);
      if (np > 1) issue_S(1);
      for (int i = 0; i < np; ++i) {
        const int st = i % kFaStages, sb = i & 1;
        if (i + 2 < np) {  // S_i done: its K stage takes page i + 2
          mbar_wait(&s_full[sb], (uint32_t)(i >> 1) & 1u);
          issue_k(i + 2);
        }
        mbar_wait(&p_full[sb], (uint32_t)(i >> 1) & 1u);  // P_i stored, O rescaled
        mbar_wait(&v_full[st], (uint32_t)(i / kFaStages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t v0 = smem_u32(sKV + st * kFaStage + 2 * kFaHalf);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // 16 positions (8 P columns) per step
          const uint64_t b = umma_desc_sw128_mn(v0 + kk * 2048, kFaHalf);
          umma_bf16_tmem_a(tO, tS(sb) + kk * 8, b, idO, (i > 0 || kk > 0) ? 1u : 0u);
          umma_bf16_tmem_a(tO, tS(sb) + 32 + kk * 8, b, idO, 1u);
        }
        umma_commit(&o_done);
        if (i + 2 < np) {
          issue_S(i + 2);  // into the buffer PV_i reads: tensor-core ops run in order
          mbar_wait(&o_done, (uint32_t)(i & 1));
          issue_v(i + 2);
        }
      }
    }
  } else {
    // ---- softmax warps: thread (r, hf) owns 32 positions of each page of row r
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const int lim = start + (row0 + r < span_rows ? row0 + r : span_rows - 1) / G;
    float m = -INFINITY, l = 0.f;  // l: this half's share of the row sum
    for (int i = 0; i < np; ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (uint32_t)(i >> 1) & 1u);
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float s[32];
      tmem_ld32(tS(sb) + lane_off + 32 * hf, s);
      const int p0 = (t_lo + i) * kPage + 32 * hf;
      if (p0 + 31 > lim) {  // causal edge (or rows past the end): mask
#pragma unroll
        for (int e = 0; e < 32; ++e)
          if (p0 + e > lim) s[e] = -INFINITY;
      }
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 32; ++e) mx = fmaxf(mx, s[e]);
      xch[sb][hf][r] = mx;
      named_barrier_sync(1, kFaSoftmaxWarps * 32);
      mx = fmaxf(mx, xch[sb][hf ^ 1][r]);
      // Lazy rescaling: the exponent base m moves only when the row max
      // exceeds it by more than kFaLazy (P stays <= 2^kFaLazy, harmless in
      // fp32 and in the bf16 hi/lo pair), so O in TMEM is rarely rescaled --
      // a rescale reads and writes 64 KB of TMEM per page.  l, O and the split
      // partial's m all use the same base, so the result is unchanged.
      const float mxs = mx * kFaScaleLog2;
      float alpha = 1.f;
      if (mxs > m + kFaLazy) {  // also the first finite max (m = -inf)
        alpha = exp2_ftz(m - mxs);  // 0 while nothing was seen
        m = mxs;
      }
      const float bse = m == -INFINITY ? 0.f : m;
      float rs = 0.f;
      float hi[16], lo[16];  // bf16x2 bit patterns
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        const float e0 = exp2_ftz(fmaf(s[e], kFaScaleLog2, -bse));
        const float e1 = exp2_ftz(fmaf(s[e + 1], kFaScaleLog2, -bse));
        rs += e0 + e1;
        const uint32_t h = f2_to_bf2(e0, e1);
        const float2 hv = bf2_to_f2(h);
        hi[e >> 1] = __uint_as_float(h);
        lo[e >> 1] = __uint_as_float(f2_to_bf2(e0 - hv.x, e1 - hv.y));
      }
      l = l * alpha + rs;
      if (i > 0) {  // PV_{i-1} done before O is rescaled
        mbar_wait(&o_done, (uint32_t)((i - 1) & 1));
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (__any_sync(0xffffffffu, alpha != 1.f)) {  // rescale this half's 64 dims of O
#pragma unroll
          for (int c = 0; c < 64; c += 32) {
            float o[32];
            tmem_ld32(tO + lane_off + 64 * hf + c, o);
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] *= alpha;
            tmem_st32(tO + lane_off + 64 * hf + c, o);
          }
        }
      }
      // P_i overwrites S_i in tensor memory: hi in columns 0-31, lo in 32-63
      // (bf16 pairs; this half owns 16 of each)
      tmem_st16(tS(sb) + lane_off + 16 * hf, hi);
      tmem_st16(tS(sb) + lane_off + 32 + 16 * hf, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&p_full[sb]);
    }

    // ---- epilogue: row r, dims 64*hf .. 64*hf+63 ----
    xch[0][hf][r] = l;
    if (np > 0) {
      mbar_wait(&o_done, (uint32_t)((np - 1) & 1));
      __syncwarp();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    named_barrier_sync(1, kFaSoftmaxWarps * 32);
    l += xch[0][hf ^ 1][r];
    const int rr = grow0 + row0 + r;  // global query row
    const size_t part_stride = kHeadDim + 2;
    float* prow = nullptr;  // this row's (m, l) slot of the split partials
    if (r < rows_here && nsplit > 1)
      prow = p.part + ((size_t)rr * nsplit + split) * part_stride +
             (size_t)g * M_rows * nsplit * part_stride;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    // O rows leave TMEM one per thread; they are staged through the (now idle)
    // Q and K/V buffers so that each warp stores whole rows (coalesced)
    float* stage = reinterpret_cast<float*>(sQ);  // [128 rows][kStageLd] fp32
#pragma unroll
    for (int c = 64 * hf; c < 64 * hf + 64; c += 32) {
      float o[32];
      if (np > 0) {
        tmem_ld32(tO + lane_off + c, o);  // warp-collective: every lane takes part
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] = 0.f;  // empty split: (m, l, O) = (-inf, 0, 0)
      }
      const float sc = nsplit == 1 ? inv : 1.f;
#pragma unroll
      for (int e = 0; e < 32; e += 4)
        *reinterpret_cast<float4*>(stage + r * kStageLd + c + e) =
            make_float4(o[e] * sc, o[e + 1] * sc, o[e + 2] * sc, o[e + 3] * sc);
    }
    named_barrier_sync(1, kFaSoftmaxWarps * 32);
    const int lane = tid & 31;
    for (int row = warp; row < rows_here; row += kFaSoftmaxWarps) {
      const int rw = grow0 + row0 + row;  // global query row
      const float* src = stage + row * kStageLd;
      if (nsplit == 1) {
        const int tok = rw / G, j = rw % G;
        __nv_bfloat16* o =
            p.out + (size_t)tok * p.n_heads * kHeadDim + (size_t)(g * G + j) * kHeadDim;
        const float4 v = *reinterpret_cast<const float4*>(src + 4 * lane);
        *reinterpret_cast<uint2*>(o + 4 * lane) = make_uint2(f2_to_bf2(v.x, v.y), f2_to_bf2(v.z, v.w));
      } else {
        float* dst = p.part + ((size_t)rw * nsplit + split) * part_stride +
                     (size_t)g * M_rows * nsplit * part_stride;
#pragma unroll
        for (int h = 0; h < 2; ++h)  // rows are 520 B apart: 8-B stores
          *reinterpret_cast<float2*>(dst + 64 * h + 2 * lane) =
              *reinterpret_cast<const float2*>(src + 64 * h + 2 * lane);
      }
    }
    if (prow && hf == 0) {
      prow[kHeadDim] = m;
      prow[kHeadDim + 1] = l;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

int attn_umma_splits(int n_kv, int q_tiles, int T, int num_sms) {
  const int tiles = (T + kPage - 1) / kPage;
  static const int cap = [] {  // tuning knob: most KV splits per query tile
    const char* e = getenv("SR_ATTN_SPLITS_MAX");
    const int v = e ? atoi(e) : 8;  // 8 vs 16: 4.37 vs 4.48 ms (7B, M = 80, 2 K context)
    return v < 1 ? 1 : v > 16 ? 16 : v;
  }();
  int s = 2 * num_sms / (n_kv * q_tiles);  // two CTAs per SM
  if (s > tiles) s = tiles;
  if (s > cap) s = cap;
  return s < 1 ? 1 : s;
}

int attn_umma_q_tiles(int M_tokens, int G) { return (M_tokens * G + kFaRows - 1) / kFaRows; }

cudaError_t attn_umma_launch(const void* tmK, const void* tmV, const AttnParams& p, int M_tokens,
                             int nsplit, cudaStream_t stream, int n_items) {
  const int G = p.n_heads / p.n_kv;
  const int M_rows = M_tokens * G;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_prefill_umma_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kFaSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_kv, nsplit, p.spans ? n_items : (M_rows + kFaRows - 1) / kFaRows);
  cfg.blockDim = dim3(kFaThreads);
  cfg.dynamicSmemBytes = kFaSmem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, attn_prefill_umma_kernel, *(const CUtensorMap*)tmK,
                            *(const CUtensorMap*)tmV, p, M_rows, G);
}

}  // namespace sr
