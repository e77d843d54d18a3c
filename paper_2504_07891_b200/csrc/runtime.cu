// Native runtime behind the C-ABI (include/specreason_b200.h).
//
// A model handle carves the caller's workspace into activation buffers and a
// DecodeState, and owns one CUDA graph per model:
//
//   [cond_init] -> WHILE(cond) { layer 0..L-1: qkv GEMV | attention | o GEMV |
//                                gate/up GEMV | down GEMV ;  LM-head argmax }
//
// The LM-head kernel's last CTA chooses the token, runs the stop test and sets
// the while-condition from the device (cudaGraphSetConditional), so a whole
// step's decode is one graph launch with no host round trip per token (K10).
// Kernels inside the body are chained with programmatic dependent launch, so
// each GEMV's weight prefetch overlaps its predecessor's tail.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <string>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace sr {

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define SR_CK(expr)                                                                      \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail((int)_e, std::string(#expr) + ": " + cudaGetErrorString(_e));         \
  } while (0)

constexpr int kPrefillSplitsMax = 8;
constexpr int kAttnPrefillSplit = 16;
constexpr int kAttnItemsMax = 4096;  // (span, query tile) items of one multi-sequence pass

struct Layout {  // workspace carve-up (byte offsets)
  size_t st, h, x, q, attn, act, part, apart, actr, lm_v1, lm_v2, lm_i1, lm_ctr, logits, ro_cnt,
      mk_maps, mk_layers, mk_tiles, mk_h, mk_part, mk_apart, mk_lm, mk_prof, mk_ctab, tp_delta, tp_small, attn_items, attn_tabs,
      total;
  int mk_maxj;
  int mk_g;  // CTAs of the persistent decode kernel
  int nsplit_decode;
  size_t part_floats;
};

static size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// CTAs of the persistent decode kernel: one per SM unless SR_MK_CTAS (read
// when the model's workspace is sized and created) asks for fewer -- an
// experiment knob, and how tensor-parallel ranks sharing one GPU in a test
// leave each other room to be co-resident
static int mk_ctas_for(int num_sms) {
  const char* e = getenv("SR_MK_CTAS");
  const int v = e ? atoi(e) : 0;
  return v >= 16 && v < num_sms ? v : num_sms;
}

static Layout make_layout(const sr_model_desc& d, int num_sms) {
  Layout L{};
  const size_t T = d.max_tokens;
  const size_t qd = (size_t)d.n_heads * SR_HEAD_DIM;
  const size_t qkv = qd + 2 * (size_t)d.n_kv_heads * SR_HEAD_DIM;
  const size_t nmax = std::max<size_t>({qkv, (size_t)d.d_model, 2 * (size_t)d.d_ffn});
  L.nsplit_decode = attn_decode_splits(d.n_kv_heads, num_sms);
  const size_t nsplit_max = std::max<size_t>(L.nsplit_decode, kAttnPrefillSplit);
  const size_t lm_parts = (size_t)gemv_max_grid(num_sms) + 64;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
  L.st = take(sizeof(DecodeState));
  L.h = take(T * d.d_model * 4);
  L.x = take(T * std::max<size_t>(d.d_model, qd) * 2);
  L.q = take(T * qd * 2);
  L.attn = take(T * qd * 2);
  L.act = take(T * d.d_ffn * 2);
  // split-K partials: up to 8 splits for short (verify-sized) chunks; long
  // chunks have enough output tiles for one split (gemm() lowers the count)
  L.part_floats = (size_t)std::max<size_t>((size_t)kPrefillSplitsMax * std::min<size_t>(T, 256), T) * nmax;
  L.part = take(L.part_floats * 4);
  L.apart = take(T * d.n_heads * nsplit_max * (SR_HEAD_DIM + 2) * 4);
  L.actr = take(T * d.n_kv_heads * 4);
  L.lm_v1 = take(lm_parts * 4);
  L.lm_v2 = take(lm_parts * 4);
  L.lm_i1 = take(lm_parts * 4);
  L.lm_ctr = take(64);
  L.logits = take((size_t)d.vocab_rows * 4);
  L.ro_cnt = take(64);
  // persistent decode kernel (decode_mk.cu)
  const int mk_g = mk_ctas_for(num_sms);
  L.mk_g = mk_g;
  const int qd_i = d.n_heads * SR_HEAD_DIM, qkv_i = qd_i + 2 * d.n_kv_heads * SR_HEAD_DIM;
  L.mk_maxj = std::max({mk_max_j(qkv_i, d.d_model, mk_g), mk_max_j(d.d_model, qd_i, mk_g),
                        mk_max_j(d.d_model, d.d_ffn, mk_g)});
  L.mk_maps = take(((size_t)d.n_layers * 4 + 3) * sizeof(CUtensorMap));  // + K, V pools
  L.mk_layers = take((size_t)d.n_layers * sizeof(MkLayer));
  L.mk_tiles = take(((size_t)d.n_layers * 4 + 1) * sizeof(void*));  // tile-major weight pointers
  L.mk_h = take(2 * (size_t)d.d_model * 4);
  L.mk_part = take(3 * (size_t)mk_g * L.mk_maxj * mk_tile_rows() * 4);
  L.mk_apart = take((size_t)num_sms * 8 * 130 * 4);
  L.mk_lm = take((size_t)num_sms * 3 * 4);
  L.mk_prof = take((size_t)SR_PROF_EVENTS * 8);
  L.attn_items = take((size_t)kAttnItemsMax * 16);  // int4 per (span, query tile)
  L.attn_tabs = take((size_t)kAttnItemsMax * 8);    // page table pointer per item
  L.mk_ctab = take(3 * 256 * 2 + 64 * 4);
  // tensor parallelism: the all-reduced row-parallel output, exchange buffers
  L.tp_delta = take(T * d.d_model * 4);
  L.tp_small = take(4096 + 4 * 8192);  // exchange words + the decode delta row
  L.total = o;
  return L;
}

struct Model {
  sr_model_desc d;
  std::vector<sr_layer_ptrs> layers;
  const __nv_bfloat16 *embed, *ln_f, *lm_head;
  const float* rope;
  __nv_bfloat16 *k_pool, *v_pool;
  Layout L;
  char* ws;
  int num_sms;
  int q_dim, kv_dim, qkv_rows;
  DecodeState* st;
  float* h;
  __nv_bfloat16 *x, *q, *attn, *act;
  float *part, *apart, *lm_v1, *lm_v2, *logits;
  int* lm_i1;
  unsigned *actr, *lm_ctr, *ro_cnt;
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  sr_timing timing{};
  bool pdl = true;
  bool stream_decode = false;  // SR_DECODE=stream: per-token host loop (profiling only)
  bool graph_decode = false;   // SR_DECODE=graph: per-kernel decode graph (A/B reference)
  MkParams mk{};
  int* trace_host = nullptr;
  void* tp_comm = nullptr;  // sr_model_set_tp (NCCL); non-null: the TP code paths run
  PeerComm* tp_peer = nullptr;  // sr_model_set_tp_peer (NVLink peer memory)
  bool tp_on() const { return tp_comm || tp_peer; }
  float* tp_delta = nullptr;
  float *tp_send, *tp_gather, *tp_dig, *tp_dec;
  int* tp_counts;
  bool prefetch = false;       // SR_PREFETCH=1: GEMV L2 prefetch before the PDL wait
  bool feed1 = true;           // one fed token decodes in the persistent kernel (SR_FEED1=0: prefill)
  struct alignas(64) TMap { CUtensorMap m; };
  std::vector<TMap> wmaps;     // per layer: qkv, o, gu, d ; then lm_head
  TMap amaps[3][5];            // [x | attn | act][token tile 32/64/96/128/256]
  TMap kvmaps[2];              // K / V pools as [L*n_pages*n_kv*64, 128], 64x64 boxes
  enum { ACT_X = 0, ACT_ATTN = 1, ACT_ACT = 2 };

  int build_tmaps() {
    wmaps.resize((size_t)d.n_layers * 4 + 1);
    for (int l = 0; l < d.n_layers; ++l) {
      const void* w[4] = {lw(l, WQKV), lw(l, WO), lw(l, WGU), lw(l, WD)};
      const int rows[4] = {qkv_rows, d.d_model, 2 * d.d_ffn, d.d_model};
      const int cols[4] = {d.d_model, q_dim, d.d_model, d.d_ffn};
      for (int i = 0; i < 4; ++i)
        if (make_tmap_bf16(&wmaps[l * 4 + i].m, w[i], rows[i], cols[i], 128))
          return fail(SR_E_INVALID, "cuTensorMapEncodeTiled failed for a weight");
    }
    if (make_tmap_bf16(&wmaps.back().m, lm_head, d.vocab_rows, d.d_model, 128))
      return fail(SR_E_INVALID, "cuTensorMapEncodeTiled failed for lm_head");
    const void* a[3] = {x, attn, act};
    const int acols[3] = {d.d_model, q_dim, d.d_ffn};
    const int tiles[5] = {32, 64, 96, 128, 256};
    for (int i = 0; i < 3; ++i)
      for (int t = 0; t < 5; ++t)
        if (make_tmap_bf16(&amaps[i][t].m, a[i], d.max_tokens, acols[i], tiles[t]))
          return fail(SR_E_INVALID, "cuTensorMapEncodeTiled failed for an activation");
    const long kv_rows = (long)d.n_layers * d.n_pages * d.n_kv_heads * SR_PAGE;
    if (kv_rows >= (1L << 31)) return fail(SR_E_INVALID, "K/V pool too large for a tensor map");
    const void* pools[2] = {k_pool, v_pool};
    for (int i = 0; i < 2; ++i)
      if (make_tmap_bf16_box(&kvmaps[i].m, pools[i], (int)kv_rows, SR_HEAD_DIM, 64, SR_PAGE, true))
        return fail(SR_E_INVALID, "cuTensorMapEncodeTiled failed for a K/V pool");
    return 0;
  }

  // tensor maps (32-row x 256-col boxes, no swizzle) + per-layer table for the
  // persistent decode kernel, written into the workspace once
  int build_mk() {
    const int n = d.n_layers * 4 + 1;
    std::vector<TMap> maps(n + 2);
    maps[n] = kvmaps[0];  // K / V pools, 64 x 64 boxes, 128-B swizzle (decode attention)
    maps[n + 1] = kvmaps[1];
    for (int l = 0; l < d.n_layers; ++l) {
      const void* w[4] = {lw(l, WQKV), lw(l, WO), lw(l, WGU), lw(l, WD)};
      const int rows[4] = {qkv_rows, d.d_model, 2 * d.d_ffn, d.d_model};
      const int cols[4] = {d.d_model, q_dim, d.d_model, d.d_ffn};
      for (int i = 0; i < 4; ++i)
        if (make_tmap_bf16_box(&maps[l * 4 + i].m, w[i], rows[i], cols[i],
                               std::min(cols[i], mk_tile_cols()), mk_tile_rows(), false))
          return fail(SR_E_INVALID, "cuTensorMapEncodeTiled failed for a decode weight map");
    }
    if (make_tmap_bf16_box(&maps[n - 1].m, lm_head, d.vocab_rows, d.d_model,
                           std::min(d.d_model, mk_tile_cols()), mk_tile_rows(), false))
      return fail(SR_E_INVALID, "cuTensorMapEncodeTiled failed for the LM-head map");
    // contributor tables of the tile-range phases (same partition as the kernel)
    {
      const int N3[3] = {qkv_rows, d.d_model, d.d_model};
      const int K3[3] = {d.d_model, q_dim, d.d_ffn};
      std::vector<uint16_t> tab(3 * 256, 0);
      const long G = L.mk_g;
      if (G > 255) return fail(SR_E_INVALID, "decode tables assume <= 255 SMs");
      for (int t = 0; t < 3; ++t) {
        const int tcol = std::min(K3[t], mk_tile_cols());
        const long kt = (K3[t] + tcol - 1) / tcol, nb = (N3[t] + 31) / 32, T = kt * nb;
        if (nb > 256) return fail(SR_E_INVALID, "decode tables hold <= 256 row blocks");
        for (long b = 0; b < nb; ++b) {
          const long u0 = b * kt, u1 = u0 + kt - 1;
          // owner of unit u / first unit of CTA c under the kernel's partition
          auto owner = [&](long u) { return T >= G ? ((u + 1) * G - 1) / T : u; };
          auto first = [&](long c) { return T >= G ? T * c / G : std::min(c, T); };
          const long c0 = owner(u0), c1 = owner(u1);
          const long j0 = b - first(c0) / kt;
          if (j0 >= L.mk_maxj || j0 > 15 || c1 - c0 + 1 > 8)
            return fail(SR_E_INVALID, "decode partial tables out of range");
          tab[t * 256 + b] = (uint16_t)(c0 | (c1 - c0 + 1) << 8 | j0 << 12);
        }
      }
      SR_CK(cudaMemcpy(ws + L.mk_ctab, tab.data(), tab.size() * 2, cudaMemcpyHostToDevice));
      mk.ctab = at<const uint16_t>(L.mk_ctab);
      mk.attn_cnt = at<int>(L.mk_ctab + 3 * 256 * 2);
    }
    std::vector<MkLayer> ly(d.n_layers);
    for (int l = 0; l < d.n_layers; ++l) ly[l] = MkLayer{lw(l, LN1), lw(l, BQKV), lw(l, LN2), nullptr};
    SR_CK(cudaMemcpy(ws + L.mk_maps, maps.data(), (n + 2) * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
    SR_CK(cudaMemcpy(ws + L.mk_layers, ly.data(), ly.size() * sizeof(MkLayer),
                     cudaMemcpyHostToDevice));
    MkParams& p = mk;
    p.maps = at<const CUtensorMap>(L.mk_maps);
    p.layers = at<const MkLayer>(L.mk_layers);
    p.embed = embed;
    p.ln_f = ln_f;
    p.rope = rope;
    p.k_pool = k_pool;
    p.v_pool = v_pool;
    p.hA = at<float>(L.mk_h);
    p.hB = p.hA + d.d_model;
    const size_t pstride = (size_t)L.mk_g * L.mk_maxj * mk_tile_rows();
    p.part_qkv = at<float>(L.mk_part);
    p.part_o = p.part_qkv + pstride;
    p.part_d = p.part_o + pstride;
    p.apart = at<float>(L.mk_apart);
    p.lm_part = at<float>(L.mk_lm);
    p.act = act;
    p.attn = attn;
    p.st = st;
    const char* pe = getenv("SR_MK_PROF");
    p.prof = (pe && pe[0] == '1') ? at<unsigned long long>(L.mk_prof) : nullptr;
    const char* te = getenv("SR_MK_TRACE");
    p.trace = nullptr;
    if (te && te[0] == '1') {  // bring-up aid: progress words readable after a hang
      SR_CK(cudaHostAlloc((void**)&trace_host, (size_t)num_sms * 8 * 4, cudaHostAllocMapped));
      memset(trace_host, 0, (size_t)num_sms * 8 * 4);
      int* dptr = nullptr;
      SR_CK(cudaHostGetDevicePointer((void**)&dptr, trace_host, 0));
      p.trace = dptr;
    }
    p.L = d.n_layers;
    p.d = d.d_model;
    p.H = d.n_heads;
    p.KV = d.n_kv_heads;
    p.f = d.d_ffn;
    p.vocab_rows = d.vocab_rows;
    p.vocab_text = d.vocab_text;
    p.n_pages = d.n_pages;
    p.q_dim = q_dim;
    p.kv_dim = kv_dim;
    p.qkv_rows = qkv_rows;
    p.eps = d.rms_eps;
    p.maxj = L.mk_maxj;
    const int tc = mk_tile_cols();
    p.xs_elems = (std::max({d.d_model, q_dim, d.d_ffn}) + tc - 1) / tc * tc;
    p.stages = mk_pick_stages(p.xs_elems);
    p.kv_dbl = mk_pick_kv_dbl(p.stages, p.xs_elems);
    if (const char* v = getenv("SR_MK_KVDBL")) p.kv_dbl = p.kv_dbl && atoi(v) != 0;
    p.tiles = nullptr;
    p.tiled = 0;
    p.vec_prologue = 1;
    if (const char* v = getenv("SR_MK_VECPRO")) p.vec_prologue = atoi(v);
    // L2 prefetch run-ahead beyond the ring (tiles of the decode-layout copy).
    // Measured (round 2, same box): 4-8 tiles speed up the chain-bound 1.5B by
    // 2 % (1.077 -> 1.056 ms/token at 2 K); any run-ahead slows the HBM-bound
    // 32B (10.89 -> 11.24 / 11.92 at 8 / 16 tiles).  On for models whose
    // layer streams < 256 MB (the draft), off otherwise.
    {
      const double layer_bytes = 2.0 * ((double)qkv_rows * d.d_model + (double)d.d_model * q_dim +
                                        3.0 * d.d_model * d.d_ffn);
      p.l2_ahead = layer_bytes < 256e6 ? 4 : -1;
    }
    if (const char* v = getenv("SR_MK_L2AHEAD")) p.l2_ahead = atoi(v);
    p.head_split = 0;  // SR_MK_HEADSPLIT=1: split a page's heads over idle CTAs (round 1; no gain with the tensor-core attention)
    if (const char* v = getenv("SR_MK_HEADSPLIT")) p.head_split = atoi(v);
    p.combine_wide = -1;  // SR_MK_COMBW=0/1: A/B of the 64-dim COMBINE items
    if (const char* v = getenv("SR_MK_COMBW")) p.combine_wide = atoi(v);
    p.bar_sleep = 0;
    p.evict_first = 1;
    p.min_pages = 1;
    if (const char* v = getenv("SR_MK_MINPAGES")) p.min_pages = std::max(1, atoi(v));
    if (const char* v = getenv("SR_MK_EVICT_FIRST")) p.evict_first = atoi(v);
    if (const char* v = getenv("SR_MK_BARSLEEP")) p.bar_sleep = atoi(v);
    p.no_load = 0;
    if (const char* v = getenv("SR_MK_NOLOAD")) p.no_load = atoi(v);
    return 0;
  }

  template <typename T>
  T* at(size_t off) { return reinterpret_cast<T*>(ws + off); }

  const __nv_bfloat16* lw(int l, int which) const {
    const sr_layer_ptrs& p = layers[l];
    const void* v[] = {p.ln1, p.wqkv, p.bqkv, p.wo, p.ln2, p.wgu, p.wd};
    return reinterpret_cast<const __nv_bfloat16*>(v[which]);
  }
  enum { LN1, WQKV, BQKV, WO, LN2, WGU, WD };

  GemvParams gemv_base() const {
    GemvParams p{};
    p.eps = d.rms_eps;
    p.rope = rope;
    p.k_pool = k_pool;
    p.v_pool = v_pool;
    p.n_pages = d.n_pages;
    p.n_kv = d.n_kv_heads;
    p.q_dim = q_dim;
    p.kv_dim = kv_dim;
    p.h = h;
    p.st = st;
    p.prefetch = prefetch ? 1 : 0;
    return p;
  }

  // ------------------------------------------------------- decode step ----
  cudaError_t enqueue_decode_step(cudaStream_t s) {
    cudaError_t e;
    for (int l = 0; l < d.n_layers; ++l) {
      GemvParams p = gemv_base();
      p.layer = l;
      p.W = lw(l, WQKV);
      p.N = qkv_rows;
      p.K = d.d_model;
      p.norm_w = lw(l, LN1);
      p.bias = lw(l, BQKV);
      p.embed = embed;
      p.qout = q;
      e = gemv_launch(l == 0 ? GEMV_QKV_EMBED : GEMV_QKV, p, num_sms, s, pdl && l > 0);
      if (e != cudaSuccess) return e;

      AttnParams a{};
      a.q = q;
      a.out = attn;
      a.k_pool = k_pool;
      a.v_pool = v_pool;
      a.part = apart;
      a.counters = actr;
      a.layer = l;
      a.n_pages = d.n_pages;
      a.n_heads = d.n_heads;
      a.n_kv = d.n_kv_heads;
      a.nsplit = L.nsplit_decode;
      a.st = st;
      e = attn_decode_tc_launch(a, s, pdl);
      if (e != cudaSuccess) return e;

      p = gemv_base();
      p.W = lw(l, WO);
      p.N = d.d_model;
      p.K = q_dim;
      p.x = attn;
      e = gemv_launch(GEMV_RESID, p, num_sms, s, pdl);
      if (e != cudaSuccess) return e;

      p = gemv_base();
      p.W = lw(l, WGU);
      p.N = 2 * d.d_ffn;
      p.K = d.d_model;
      p.norm_w = lw(l, LN2);
      p.act_out = act;
      e = gemv_launch(GEMV_GLU, p, num_sms, s, pdl);
      if (e != cudaSuccess) return e;

      p = gemv_base();
      p.W = lw(l, WD);
      p.N = d.d_model;
      p.K = d.d_ffn;
      p.x = act;
      e = gemv_launch(GEMV_RESID, p, num_sms, s, pdl);
      if (e != cudaSuccess) return e;
    }
    GemvParams p = gemv_base();
    p.W = lm_head;
    p.N = d.vocab_rows;
    p.K = d.d_model;
    p.n_valid = d.vocab_text;
    p.norm_w = ln_f;
    p.part_v1 = lm_v1;
    p.part_v2 = lm_v2;
    p.part_i1 = lm_i1;
    p.counter = lm_ctr;
    return gemv_launch(GEMV_LM_ARGMAX, p, num_sms, s, pdl);
  }

  int build_graph() {
    SR_CK(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
    SR_CK(cudaGraphCreate(&graph, 0));
    SR_CK(cudaGraphConditionalHandleCreate(&cond, graph, 0, 0));
    SR_CK(cudaStreamBeginCaptureToGraph(cap_stream, graph, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed));
    cudaError_t e = cond_init_launch(st, (unsigned long long)cond, cap_stream);
    cudaGraph_t g2 = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap_stream, &g2);
    SR_CK(e);
    SR_CK(e2);
    size_t n = 0;
    SR_CK(cudaGraphGetNodes(graph, nullptr, &n));
    if (n != 1) return fail(SR_E_GRAPH, "unexpected node count in decode graph prologue");
    cudaGraphNode_t init_node;
    SR_CK(cudaGraphGetNodes(graph, &init_node, &n));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    SR_CK(cudaGraphAddNode(&cnode, graph, &init_node, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SR_CK(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed));
    e = enqueue_decode_step(cap_stream);
    e2 = cudaStreamEndCapture(cap_stream, &body);
    SR_CK(e);
    SR_CK(e2);
    SR_CK(cudaGraphInstantiate(&exec, graph, 0));
    return 0;
  }

  // ------------------------------------------------------------ prefill ---
  // One sequence's rows inside a prefill pass: rows [row0, row0 + M) sit at
  // positions start.. of the stream whose page table is `page_table`.
  struct SeqSpan {
    const int* page_table;
    int start, row0, M;
  };

  // Runs ids[0..n) at positions start.. through all layers, chunked by
  // max_tokens; leaves the final-normed rows of the last chunk in x.
  // Returns the row count of the last chunk.
  int prefill(const int* page_table, int start, const int* ids, int n, cudaStream_t s,
              int* last_rows) {
    const int T = d.max_tokens;
    int rows = 0;
    for (int c0 = 0; c0 < n; c0 += T) {
      const int M = std::min(T, n - c0);
      rows = M;
      const SeqSpan sp{page_table, start + c0, 0, M};
      if (int rc = run_layers(ids + c0, M, &sp, 1, nullptr, s)) return rc;
    }
    *last_rows = rows;
    return 0;
  }

  // One pass of M rows (<= max_tokens) through every layer.  The rows may
  // belong to several sequences (spans): the GEMMs and epilogues run over all
  // rows at once, attention runs per span over that span's own K/V pages.
  // tok_meta (device, (position, page) per row) is required when n_spans > 1.
  int run_layers(const int* ids, int M, const SeqSpan* spans, int n_spans, const int* tok_meta,
                 cudaStream_t s) {
    SR_CK(embed_norm_launch(ids, M, embed, d.d_model, lw(0, LN1), d.rms_eps, h, x, s));
    // several spans on the tcgen05 attention: one launch per layer over a
    // (span, query tile) item table
    const bool multi = n_spans > 1;
    int n_items = 0, t_max = 0;
    if (multi) {
      const int G = d.n_heads / d.n_kv_heads;
      std::vector<int4> items;
      std::vector<const int*> tabs;
      for (int k = 0; k < n_spans; ++k) {
        const int tiles = attn_umma_q_tiles(spans[k].M, G);
        for (int t = 0; t < tiles; ++t) {
          items.push_back(make_int4(spans[k].row0, spans[k].M, spans[k].start, t));
          tabs.push_back(spans[k].page_table);
        }
        t_max = std::max(t_max, spans[k].start + spans[k].M);
      }
      n_items = (int)items.size();
      if (n_items > kAttnItemsMax) return fail(SR_E_CAPACITY, "too many attention items");
      SR_CK(cudaMemcpyAsync(ws + L.attn_items, items.data(), items.size() * sizeof(int4),
                            cudaMemcpyHostToDevice, s));
      SR_CK(cudaMemcpyAsync(ws + L.attn_tabs, tabs.data(), tabs.size() * sizeof(const int*),
                            cudaMemcpyHostToDevice, s));
    }
    for (int l = 0; l < d.n_layers; ++l) {
      // qkv
      int rc = gemm(ACT_X, l * 4 + 0, x, lw(l, WQKV), M, qkv_rows, d.d_model, s);
      if (rc) return -rc;
      EpiParams ep = epi_base(M, qkv_rows);
      ep.bias = lw(l, BQKV);
      ep.q = q;
      ep.page_table = spans[0].page_table;
      ep.start_pos = spans[0].start;
      ep.tok_meta = tok_meta;
      ep.layer = l;
      SR_CK(epi_qkv_launch(ep, s));
      watch(s, "qkv gemm+epi", l, M, last_splits);
      // attention: all spans in one launch, or per sequence
      if (multi) {
        AttnParams a{};
        a.q = q;
        a.out = attn;
        a.k_pool = k_pool;
        a.v_pool = v_pool;
        a.page_table = spans[0].page_table;
        a.part = apart;
        a.counters = actr;
        a.layer = l;
        a.n_pages = d.n_pages;
        a.n_heads = d.n_heads;
        a.n_kv = d.n_kv_heads;
        a.spans = reinterpret_cast<const int4*>(ws + L.attn_items);
        a.span_tables = reinterpret_cast<const int* const*>(ws + L.attn_tabs);
        a.nsplit = std::min(kAttnPrefillSplit, attn_umma_splits(d.n_kv_heads, n_items, t_max, num_sms));
        SR_CK(attn_umma_launch(&kvmaps[0].m, &kvmaps[1].m, a, M, a.nsplit, s, n_items));
        if (a.nsplit > 1) SR_CK(attn_merge_launch(a, M, a.nsplit, s));
        watch(s, "attn_prefill_umma (spans)", l, M, a.nsplit);
      }
      for (int k = 0; k < (multi ? 0 : n_spans); ++k) {
        const SeqSpan& sp = spans[k];
        AttnParams a{};
        a.q = q + (size_t)sp.row0 * q_dim;
        a.out = attn + (size_t)sp.row0 * q_dim;
        a.k_pool = k_pool;
        a.v_pool = v_pool;
        a.page_table = sp.page_table;
        a.part = apart;
        a.counters = actr;
        a.layer = l;
        a.n_pages = d.n_pages;
        a.n_heads = d.n_heads;
        a.n_kv = d.n_kv_heads;
        const int Tlast = sp.start + sp.M;
        a.start_pos = sp.start;
        a.st = nullptr;
        {
          const int G = d.n_heads / d.n_kv_heads;
          a.nsplit = std::min(kAttnPrefillSplit, attn_umma_splits(d.n_kv_heads,
                                                                  attn_umma_q_tiles(sp.M, G),
                                                                  Tlast, num_sms));
          SR_CK(attn_umma_launch(&kvmaps[0].m, &kvmaps[1].m, a, sp.M, a.nsplit, s));
          if (a.nsplit > 1) SR_CK(attn_merge_launch(a, sp.M, a.nsplit, s));
          watch(s, "attn_prefill_umma", l, sp.M, a.nsplit);
        }
      }
      // o-proj + residual + norm2
      rc = gemm(ACT_ATTN, l * 4 + 1, attn, lw(l, WO), M, d.d_model, q_dim, s);
      if (rc) return -rc;
      ep = epi_base(M, d.d_model);
      ep.norm_w = lw(l, LN2);
      if (tp_on())
        if (int rc2 = tp_reduce_rows(ep, M, s)) return -rc2;
      SR_CK(epi_resid_norm_launch(ep, s));
      // gate/up
      rc = gemm(ACT_X, l * 4 + 2, x, lw(l, WGU), M, 2 * d.d_ffn, d.d_model, s, act);
      if (rc) return -rc;
      if (!fused_glu) {
        ep = epi_base(M, 2 * d.d_ffn);
        SR_CK(epi_glu_launch(ep, s));
      }
      watch(s, "o/gu gemm+epi", l, M, last_splits);
      // down + residual + next norm
      rc = gemm(ACT_ACT, l * 4 + 3, act, lw(l, WD), M, d.d_model, d.d_ffn, s);
      if (rc) return -rc;
      ep = epi_base(M, d.d_model);
      ep.norm_w = (l + 1 < d.n_layers) ? lw(l + 1, LN1) : ln_f;
      if (tp_on())
        if (int rc2 = tp_reduce_rows(ep, M, s)) return -rc2;
      SR_CK(epi_resid_norm_launch(ep, s));
    }
    return 0;
  }

  // ----------------------------------------------------- tensor parallel ---
  int tp_check(int r, const char* what) {
    if (r != 0) return fail(SR_E_TP, std::string(what) + ": " + tp_error_string(r));
    return 0;
  }

  // host-driven collectives: NCCL when a communicator is attached (ring
  // algorithms for the large prefill deltas), else the peer-memory one-shot
  int peer_check(int r, const char* what) {
    if (r != 0) return fail(SR_E_TP, std::string(what) + ": peer exchange failed (" +
                                         std::to_string(r) + ")");
    return 0;
  }
  int coll_all_reduce_f32(float* buf, size_t n, cudaStream_t s) {
    if (tp_comm) return tp_check(tp_all_reduce_f32(tp_comm, buf, n, s), "ncclAllReduce");
    return peer_check(peer_exchange(tp_peer, 0, buf, buf, n, 0, s), "all-reduce");
  }
  int coll_all_reduce_i32(int* buf, size_t n, cudaStream_t s) {
    if (tp_comm) return tp_check(tp_all_reduce_i32(tp_comm, buf, n, s), "ncclAllReduce");
    return peer_check(peer_exchange(tp_peer, 3, reinterpret_cast<float*>(buf),
                                    reinterpret_cast<float*>(buf), n, 0, s), "all-reduce");
  }
  int coll_all_gather_f32(const float* send, float* recv, size_t n, cudaStream_t s) {
    if (tp_comm) return tp_check(tp_all_gather_f32(tp_comm, send, recv, n, s), "ncclAllGather");
    return peer_check(peer_exchange(tp_peer, 1, send, recv, n, 0, s), "all-gather");
  }
  int coll_broadcast_f32(const float* send, float* recv, size_t n, int root, cudaStream_t s) {
    if (tp_comm) return tp_check(tp_broadcast_f32(tp_comm, send, recv, n, root, s), "ncclBroadcast");
    return peer_check(peer_exchange(tp_peer, 2, send, recv, n, root, s), "broadcast");
  }

  // prefill: all-reduce the row-parallel output (split partials -> delta)
  // and point the residual epilogue at it
  int tp_reduce_rows(EpiParams& ep, int M, cudaStream_t s) {
    const size_t n = (size_t)M * d.d_model;
    SR_CK(split_sum_launch(part, ep.splits, (size_t)M * d.d_model, tp_delta, n, s));
    if (int rc = coll_all_reduce_f32(tp_delta, n, s)) return rc;
    ep.part = tp_delta;
    ep.splits = 1;
    return 0;
  }

  // greedy step over vocab-parallel logits (local rows in `logits`)
  int tp_select(cudaStream_t s) {
    const int grid = std::min(gemv_max_grid(num_sms), (d.vocab_text + 255) / 256);
    SR_CK(tp_top2_local_launch(logits, d.vocab_text, d.vocab_base, lm_v1, lm_v2, lm_i1, lm_ctr,
                               tp_send, std::max(grid, 1), s));
    if (int rc = coll_all_gather_f32(tp_send, tp_gather, 3, s)) return rc;
    SR_CK(tp_select_launch(tp_gather, d.tp_world, st, s));
    return 0;
  }

  // one decoded token with the TP exchanges (host-driven loop)
  int tp_decode_step(cudaStream_t s) {
    for (int l = 0; l < d.n_layers; ++l) {
      GemvParams p = gemv_base();
      p.layer = l;
      p.W = lw(l, WQKV);
      p.N = qkv_rows;
      p.K = d.d_model;
      p.norm_w = lw(l, LN1);
      p.bias = lw(l, BQKV);
      p.embed = embed;
      p.qout = q;
      SR_CK(gemv_launch(l == 0 ? GEMV_QKV_EMBED : GEMV_QKV, p, num_sms, s, false));
      AttnParams a{};
      a.q = q;
      a.out = attn;
      a.k_pool = k_pool;
      a.v_pool = v_pool;
      a.part = apart;
      a.counters = actr;
      a.layer = l;
      a.n_pages = d.n_pages;
      a.n_heads = d.n_heads;
      a.n_kv = d.n_kv_heads;
      a.nsplit = L.nsplit_decode;
      a.st = st;
      SR_CK(attn_decode_tc_launch(a, s, false));
      for (int half = 0; half < 2; ++half) {
        p = gemv_base();
        if (half == 0) {  // o-proj (row parallel) -> delta
          p.W = lw(l, WO);
          p.N = d.d_model;
          p.K = q_dim;
          p.x = attn;
        } else {          // gate/up, then down (row parallel) -> delta
          GemvParams g = gemv_base();
          g.W = lw(l, WGU);
          g.N = 2 * d.d_ffn;
          g.K = d.d_model;
          g.norm_w = lw(l, LN2);
          g.act_out = act;
          SR_CK(gemv_launch(GEMV_GLU, g, num_sms, s, false));
          p.W = lw(l, WD);
          p.N = d.d_model;
          p.K = d.d_ffn;
          p.x = act;
        }
        p.h = tp_dec;  // zero on entry; the residual GEMV adds into it
        SR_CK(gemv_launch(GEMV_RESID, p, num_sms, s, false));
        if (int rc = tp_check(tp_all_reduce_f32(tp_comm, tp_dec, d.d_model, s), "ncclAllReduce"))
          return rc;
        SR_CK(add_delta_launch(h, tp_dec, d.d_model, s));
      }
    }
    GemvParams p = gemv_base();
    p.W = lm_head;
    p.N = d.vocab_rows;
    p.K = d.d_model;
    p.norm_w = ln_f;
    p.logits = logits;
    SR_CK(gemv_launch(GEMV_LM_LOGITS, p, num_sms, s, false));
    return tp_select(s);
  }

  int last_splits = 1;
  bool fused_glu = false;  // the last gemm() wrote silu(gate)*up itself
  // SR_ATTN_PHI=1: prefill attention with bf16 P only.  Off: the hi/lo split
  // of P is needed for the tiny-model parity bound (measured: bf16 P fails
  // tests/test_gpu_parity.py) and costs only ~2-3 % of a verify pass
  // SR_WATCH=1: synchronise after each prefill stage and abort with the stage
  // name if it does not finish within 10 s (bring-up aid for device hangs)
  bool watch_on = false;
  int watch_ms = 10000;
  void watch(cudaStream_t s, const char* what, int layer, int M, int extra) {
    if (!watch_on) return;
    for (int i = 0; i < watch_ms; ++i) {
      cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) return;
      if (e != cudaErrorNotReady) {
        fprintf(stderr, "[sr watch] %s layer %d M %d extra %d: %s\n", what, layer, M, extra,
                cudaGetErrorString(e));
        abort();
      }
      struct timespec ts = {0, 1000000};
      nanosleep(&ts, nullptr);
    }
    fprintf(stderr, "[sr watch] HANG in %s layer %d M %d extra %d\n", what, layer, M, extra);
    abort();
  }

  int gemm(int act_id, int wmap, const __nv_bfloat16* A, const __nv_bfloat16* B, int M, int N,
           int K, cudaStream_t s, __nv_bfloat16* glu_out = nullptr) {
    fused_glu = false;
    {
      TcGemmArgs a{};
      a.act = glu_out;
      const int nt = tc_pick_tile(M, N, num_sms);
      a.nt = nt;
      const int ti = nt == 32 ? 0 : nt == 64 ? 1 : nt == 96 ? 2 : nt == 128 ? 3 : 4;
      a.tmW = &wmaps[wmap].m;
      a.tmX = &amaps[act_id][ti].m;
      a.C = part;
      a.M = M;
      a.N = N;
      a.K = K;
      int sp = tc_pick_splits(M, N, K, num_sms, nt);
      while (sp > 1 && (size_t)sp * M * N > L.part_floats) --sp;
      a.splits = sp;
      last_splits = sp;
      fused_glu = glu_out != nullptr && sp == 1;
      SR_CK(gemm_tc_launch(a, s));
      return 0;
    }
  }

  EpiParams epi_base(int M, int N) const {
    EpiParams e{};
    e.part = part;
    e.splits = last_splits;
    e.M = M;
    e.N = N;
    e.h = h;
    e.eps = d.rms_eps;
    e.x = x;
    e.rope = rope;
    e.k_pool = k_pool;
    e.v_pool = v_pool;
    e.n_pages = d.n_pages;
    e.n_kv = d.n_kv_heads;
    e.q_dim = q_dim;
    e.kv_dim = kv_dim;
    e.act = act;
    return e;
  }
};

static int validate(const sr_model_desc* d) {
  if (!d) return fail(SR_E_INVALID, "null descriptor");
  if (d->head_dim != SR_HEAD_DIM) return fail(SR_E_INVALID, "head_dim must be 128");
  if (d->n_layers < 1 || d->d_model < 128 || d->d_model % 128 != 0)
    return fail(SR_E_INVALID, "d_model must be a multiple of 128");
  if (d->n_heads % d->n_kv_heads != 0 || d->n_heads / d->n_kv_heads > 8)
    return fail(SR_E_INVALID, "unsupported GQA group");
  if (d->d_ffn % 32 != 0) return fail(SR_E_INVALID, "d_ffn must be a multiple of 32");
  if (d->vocab_text % 2 != 0 || d->vocab_rows % 2 != 0 || d->vocab_text > d->vocab_rows)
    return fail(SR_E_INVALID, "vocab sizes must be even, text <= rows");
  if (d->max_tokens < 1 || d->max_new < 1 || d->n_pages < 1 || d->max_pos < 1)
    return fail(SR_E_INVALID, "capacities must be positive");
  if (d->tp_world < 1 || d->tp_rank < 0 || d->tp_rank >= d->tp_world || d->vocab_base < 0)
    return fail(SR_E_INVALID, "bad tensor-parallel fields");
  return 0;
}

static int num_sms_of_current_device() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace sr

using namespace sr;

extern "C" {

int sr_abi_version(void) { return SR_ABI_VERSION; }

const char* sr_last_error(void) { return g_last_error.c_str(); }

size_t sr_workspace_bytes(const sr_model_desc* desc) {
  if (validate(desc)) return 0;
  return make_layout(*desc, num_sms_of_current_device()).total;
}

int sr_model_create(const sr_model_desc* desc, const sr_model_ptrs* ptrs, void* stream,
                    void** out_model) {
  if (int rc = validate(desc)) return rc;
  if (!ptrs || !out_model || !ptrs->layers || !ptrs->workspace)
    return fail(SR_E_INVALID, "null pointer in model pointers");
  Model* m = new Model();
  m->d = *desc;
  m->layers.assign(ptrs->layers, ptrs->layers + desc->n_layers);
  m->embed = (const __nv_bfloat16*)ptrs->embed;
  m->ln_f = (const __nv_bfloat16*)ptrs->ln_f;
  m->lm_head = (const __nv_bfloat16*)ptrs->lm_head;
  m->rope = ptrs->rope;
  m->k_pool = (__nv_bfloat16*)ptrs->k_pool;
  m->v_pool = (__nv_bfloat16*)ptrs->v_pool;
  m->num_sms = num_sms_of_current_device();
  m->L = make_layout(*desc, m->num_sms);
  m->ws = (char*)ptrs->workspace;
  m->q_dim = desc->n_heads * SR_HEAD_DIM;
  m->kv_dim = desc->n_kv_heads * SR_HEAD_DIM;
  m->qkv_rows = m->q_dim + 2 * m->kv_dim;
  m->st = m->at<DecodeState>(m->L.st);
  m->h = m->at<float>(m->L.h);
  m->x = m->at<__nv_bfloat16>(m->L.x);
  m->q = m->at<__nv_bfloat16>(m->L.q);
  m->attn = m->at<__nv_bfloat16>(m->L.attn);
  m->act = m->at<__nv_bfloat16>(m->L.act);
  m->part = m->at<float>(m->L.part);
  m->apart = m->at<float>(m->L.apart);
  m->actr = m->at<unsigned>(m->L.actr);
  m->lm_v1 = m->at<float>(m->L.lm_v1);
  m->lm_v2 = m->at<float>(m->L.lm_v2);
  m->lm_i1 = m->at<int>(m->L.lm_i1);
  m->lm_ctr = m->at<unsigned>(m->L.lm_ctr);
  m->logits = m->at<float>(m->L.logits);
  m->ro_cnt = m->at<unsigned>(m->L.ro_cnt);
  m->tp_delta = m->at<float>(m->L.tp_delta);
  m->tp_send = m->at<float>(m->L.tp_small);
  m->tp_dig = m->tp_send + 16;
  m->tp_counts = reinterpret_cast<int*>(m->tp_send + 32);
  m->tp_gather = m->tp_send + 64;  // [world][3], world <= 64
  m->tp_dec = m->tp_send + 1024;   // decode delta row (zero between uses)
  cudaStream_t s = (cudaStream_t)stream;
  // zero the whole workspace once: counters must start at 0
  cudaError_t e = cudaMemsetAsync(m->ws, 0, m->L.total, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    delete m;
    return fail((int)e, std::string("workspace init: ") + cudaGetErrorString(e));
  }
  for (auto& ev : m->ev) cudaEventCreate(&ev);
  if (const char* v = getenv("SR_NO_PDL")) m->pdl = (v[0] == '0');
  if (const char* v = getenv("SR_DECODE")) {
    m->stream_decode = strcmp(v, "stream") == 0;
    m->graph_decode = strcmp(v, "graph") == 0;
  }
  if (const char* v = getenv("SR_PREFETCH")) m->prefetch = v[0] == '1';
  if (const char* v = getenv("SR_FEED1")) m->feed1 = v[0] != '0';
  if (const char* v = getenv("SR_WATCH")) {
    m->watch_on = atoi(v) > 0;
    m->watch_ms = atoi(v) > 1 ? atoi(v) * 1000 : 10000;
  }
  if (int rc = m->build_tmaps()) {
    sr_model_destroy(m);
    return rc;
  }
  if (int rc = m->build_graph()) {
    sr_model_destroy(m);
    return rc;
  }
  if (int rc = m->build_mk()) {
    sr_model_destroy(m);
    return rc;
  }
  *out_model = m;
  return 0;
}

int sr_model_destroy(void* model) {
  Model* m = (Model*)model;
  if (!m) return 0;
  if (m->exec) cudaGraphExecDestroy(m->exec);
  if (m->graph) cudaGraphDestroy(m->graph);
  if (m->cap_stream) cudaStreamDestroy(m->cap_stream);
  if (m->trace_host) cudaFreeHost(m->trace_host);
  for (auto& ev : m->ev)
    if (ev) cudaEventDestroy(ev);
  delete m;
  return 0;
}

int sr_generate(void* model, const int32_t* page_table, int32_t start_pos, const int32_t* ids,
                int32_t n_ids, int32_t max_new, const uint8_t* token_class, int32_t* out,
                float* margins, void* stream) {
  Model* m = (Model*)model;
  if (!m || !page_table || !ids || !token_class || !out) return fail(SR_E_INVALID, "null argument");
  if (n_ids < 1 || max_new < 1 || start_pos < 0) return fail(SR_E_INVALID, "bad sizes");
  if (max_new > m->d.max_new) return fail(SR_E_CAPACITY, "max_new exceeds the model's max_new");
  if (m->d.tp_world > 1 && !m->tp_on()) return fail(SR_E_INVALID, "tensor-parallel model without a communicator");
  if (start_pos + n_ids + max_new > m->d.max_pos)
    return fail(SR_E_CAPACITY, "positions exceed max_pos");
  cudaStream_t s = (cudaStream_t)stream;
  DecodeState init{};
  init.pos = start_pos + n_ids - 1;
  init.ctx_len = start_pos + n_ids;
  init.max_new = max_new;
  init.page_table = page_table;
  init.token_class = token_class;
  init.out_ids = out + 2;
  init.out_hdr = out;
  init.margins = margins;
  init.cond_handle = 0;
  SR_CK(cudaEventRecord(m->ev[0], s));
  // a single fed token (the stream already holds the rest of the prompt, e.g.
  // the next step of the same generator) is a decode step: the persistent
  // kernel feeds it at start_pos and emits the first new token itself, instead
  // of a prefill pass through the GEMM path (one weight pass either way, the
  // decode kernel's at ~90 % of HBM rate)
  if (n_ids == 1 && m->feed1 && !m->tp_on() && !m->stream_decode && !m->graph_decode) {
    SR_CK(decode_begin_launch(m->st, &init, s, ids));
    SR_CK(cudaEventRecord(m->ev[1], s));
    SR_CK(mk_launch(m->mk, m->L.mk_g, s));
    SR_CK(cudaEventRecord(m->ev[2], s));
    m->timing.prefill_tokens = 0;  // tells the caller every new token was a decode step
    m->timing.decode_tokens = -1;  // filled by the caller from out[0]
    return 0;
  }
  SR_CK(decode_begin_launch(m->st, &init, s));
  int rows = 0;
  int rc = m->prefill(page_table, start_pos, ids, n_ids, s, &rows);
  if (rc) return -rc;
  // first token from the last prompt row (already final-normed in x)
  GemvParams p = m->gemv_base();
  p.W = m->lm_head;
  p.N = m->d.vocab_rows;
  p.K = m->d.d_model;
  p.n_valid = m->d.vocab_text;
  p.x = m->x + (size_t)(rows - 1) * m->d.d_model;
  p.part_v1 = m->lm_v1;
  p.part_v2 = m->lm_v2;
  p.part_i1 = m->lm_i1;
  p.counter = m->lm_ctr;
  if (m->tp_on()) {  // vocab-parallel first choice
    p.logits = m->logits;
    SR_CK(gemv_launch(GEMV_LM_LOGITS_X, p, m->num_sms, s, false));
    if (int rc2 = m->tp_select(s)) return rc2;
  } else {
    SR_CK(gemv_launch(GEMV_LM_ARGMAX_X, p, m->num_sms, s, false));
  }
  SR_CK(cudaEventRecord(m->ev[1], s));
  if (m->tp_peer) {
    // tensor parallel over peer memory: the persistent kernel decodes the
    // step, exchanging the row-parallel deltas and the greedy merge in-kernel
    SR_CK(mk_launch(m->mk, m->L.mk_g, s));
  } else if (m->tp_comm) {
    // host-driven token loop: the exchanges are NCCL calls between kernels
    for (int i = 0; i < max_new; ++i) {
      int done = 0;
      SR_CK(cudaMemcpyAsync(&done, &m->st->done, sizeof(int), cudaMemcpyDeviceToHost, s));
      SR_CK(cudaStreamSynchronize(s));
      if (done) break;
      if (int rc2 = m->tp_decode_step(s)) return rc2;
    }
  } else if (!m->stream_decode && !m->graph_decode) {
    // one persistent kernel decodes the whole step (decode_mk.cu)
    SR_CK(mk_launch(m->mk, m->L.mk_g, s));
  } else if (m->graph_decode) {
    SR_CK(cudaGraphLaunch(m->exec, s));
  } else {
    // profiling mode (SR_DECODE=stream): same kernels launched per token from
    // the host, so tools that cannot see into conditional graphs (ncu) can
    SR_CK(cudaStreamSynchronize(s));
    for (int i = 0; i < max_new; ++i) {
      int done = 0;
      SR_CK(cudaMemcpy(&done, &m->st->done, sizeof(int), cudaMemcpyDeviceToHost));
      if (done) break;
      SR_CK(m->enqueue_decode_step(s));
      SR_CK(cudaStreamSynchronize(s));
    }
  }
  SR_CK(cudaEventRecord(m->ev[2], s));
  m->timing.prefill_tokens = n_ids;
  m->timing.decode_tokens = -1;  // filled by the caller from out[0]
  return 0;
}

int sr_score(void* model, const int32_t* page_table, int32_t start_pos, const int32_t* ids,
             int32_t n_ids, const int8_t* first_digit, int32_t threshold, sr_readout* readout,
             void* stream) {
  Model* m = (Model*)model;
  if (!m || !page_table || !ids || !first_digit || !readout) return fail(SR_E_INVALID, "null argument");
  if (n_ids < 1 || start_pos < 0) return fail(SR_E_INVALID, "bad sizes");
  if (start_pos + n_ids > m->d.max_pos) return fail(SR_E_CAPACITY, "positions exceed max_pos");
  if (m->d.tp_world > 1 && !m->tp_on()) return fail(SR_E_INVALID, "tensor-parallel model without a communicator");
  cudaStream_t s = (cudaStream_t)stream;
  SR_CK(cudaEventRecord(m->ev[0], s));
  int rows = 0;
  int rc = m->prefill(page_table, start_pos, ids, n_ids, s, &rows);
  if (rc) return -rc;
  GemvParams p = m->gemv_base();
  p.st = nullptr;
  p.W = m->lm_head;
  p.N = m->d.vocab_rows;
  p.K = m->d.d_model;
  p.x = m->x + (size_t)(rows - 1) * m->d.d_model;
  p.logits = m->logits;
  SR_CK(gemv_launch(GEMV_LM_LOGITS_X, p, m->num_sms, s, false));
  if (m->tp_on()) {
    // digits 0-9 are rows of rank 0's shard: broadcast their logits, count
    // ranks locally, all-reduce the counts, all-gather the local top-2s
    if (int rc2 = m->coll_broadcast_f32(m->logits, m->tp_dig, 10, 0, s)) return rc2;
    const int grid = std::max(1, std::min(m->num_sms, (m->d.vocab_text + 255) / 256));
    SR_CK(tp_readout_local_launch(m->logits, m->d.vocab_text, m->d.vocab_base, m->tp_dig,
                                  m->tp_counts, m->lm_v1, m->lm_v2, m->lm_i1, m->lm_ctr,
                                  m->tp_send, grid, s));
    if (int rc2 = m->coll_all_reduce_i32(m->tp_counts, 10, s)) return rc2;
    if (int rc2 = m->coll_all_gather_f32(m->tp_send, m->tp_gather, 3, s)) return rc2;
    SR_CK(tp_readout_final_launch(m->tp_dig, m->tp_counts, m->tp_gather, m->d.tp_world,
                                  first_digit, threshold, readout, s));
    SR_CK(cudaEventRecord(m->ev[1], s));
    SR_CK(cudaEventRecord(m->ev[2], s));
    m->timing.prefill_tokens = n_ids;
    m->timing.decode_tokens = 0;
    return 0;
  }
  ReadoutParams r{};
  r.logits = m->logits;
  r.n_valid = m->d.vocab_text;
  r.first_digit = first_digit;
  r.threshold = threshold;
  r.counts = m->ro_cnt;
  r.part_v1 = m->lm_v1;
  r.part_v2 = m->lm_v2;
  r.part_i1 = m->lm_i1;
  r.out = readout;
  SR_CK(readout_launch(r, m->num_sms, s));
  SR_CK(cudaEventRecord(m->ev[1], s));
  SR_CK(cudaEventRecord(m->ev[2], s));
  m->timing.prefill_tokens = n_ids;
  m->timing.decode_tokens = 0;
  return 0;
}

int sr_forward_logits(void* model, const int32_t* page_table, int32_t start_pos,
                      const int32_t* ids, int32_t n_ids, int32_t all, float* logits,
                      void* stream) {
  Model* m = (Model*)model;
  if (!m || !page_table || !ids || !logits) return fail(SR_E_INVALID, "null argument");
  if (n_ids < 1 || start_pos + n_ids > m->d.max_pos) return fail(SR_E_INVALID, "bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  const int T = m->d.max_tokens;
  for (int c0 = 0; c0 < n_ids; c0 += T) {
    const int M = std::min(T, n_ids - c0);
    int rows = 0;
    int rc = m->prefill(page_table, start_pos + c0, ids + c0, M, s, &rows);
    if (rc) return -rc;
    if (all) {
      for (int r = 0; r < M; ++r) {
        GemvParams p = m->gemv_base();
        p.st = nullptr;
        p.W = m->lm_head;
        p.N = m->d.vocab_rows;
        p.K = m->d.d_model;
        p.x = m->x + (size_t)r * m->d.d_model;
        p.logits = logits + (size_t)(c0 + r) * m->d.vocab_rows;
        SR_CK(gemv_launch(GEMV_LM_LOGITS_X, p, m->num_sms, s, false));
      }
    } else if (c0 + M == n_ids) {
      GemvParams p = m->gemv_base();
      p.st = nullptr;
      p.W = m->lm_head;
      p.N = m->d.vocab_rows;
      p.K = m->d.d_model;
      p.x = m->x + (size_t)(M - 1) * m->d.d_model;
      p.logits = logits;
      SR_CK(gemv_launch(GEMV_LM_LOGITS_X, p, m->num_sms, s, false));
    }
  }
  return 0;
}

int sr_verify_tokens(void* model, const int32_t* page_table, int32_t start_pos,
                     const int32_t* ids, int32_t n_ids, int32_t* out_ids, float* margins,
                     void* stream) {
  Model* m = (Model*)model;
  if (!m || !page_table || !ids || !out_ids) return fail(SR_E_INVALID, "null argument");
  if (n_ids < 1 || start_pos < 0 || start_pos + n_ids > m->d.max_pos)
    return fail(SR_E_INVALID, "bad sizes");
  if (n_ids > m->d.max_tokens) return fail(SR_E_CAPACITY, "n_ids exceeds max_tokens");
  if (m->tp_on()) return fail(SR_E_INVALID, "sr_verify_tokens: tensor parallelism not supported");
  cudaStream_t s = (cudaStream_t)stream;
  SR_CK(cudaEventRecord(m->ev[0], s));
  int rows = 0;
  int rc = m->prefill(page_table, start_pos, ids, n_ids, s, &rows);
  if (rc) return -rc;
  // LM head for every row as one tcgen05 GEMM, then a per-row argmax
  const size_t need = (size_t)rows * m->d.vocab_rows;
  if (need > m->L.part_floats) return fail(SR_E_CAPACITY, "LM-head partials exceed the workspace");
  rc = m->gemm(Model::ACT_X, m->d.n_layers * 4, m->x, m->lm_head, rows, m->d.vocab_rows,
               m->d.d_model, s);
  if (rc) return -rc;
  SR_CK(rows_argmax_launch(m->part, m->last_splits, need, rows, m->d.vocab_rows, m->d.vocab_text,
                           m->d.vocab_base, out_ids, margins, s, m->lm_v1, m->lm_v2, m->lm_i1,
                           m->lm_ctr, gemv_max_grid(m->num_sms) + 64));
  SR_CK(cudaEventRecord(m->ev[1], s));
  SR_CK(cudaEventRecord(m->ev[2], s));
  m->timing.prefill_tokens = n_ids;
  m->timing.decode_tokens = 0;
  return 0;
}

// ------------------------------------------------------ multi-sequence ---
// Several streams' fresh rows in one pass: the GEMMs and
// epilogues run over all rows at once (one weight stream for the batch),
// attention runs per sequence, the LM head is one GEMM over each sequence's
// last row.
static constexpr int kMaxSeqs = 64;

static int batch_spans(Model* m, int32_t n_seq, const int32_t* const* page_tables,
                       const int32_t* start_pos, const int32_t* n_ids,
                       std::vector<Model::SeqSpan>& spans, int* total) {
  if (n_seq < 1 || n_seq > kMaxSeqs) return fail(SR_E_INVALID, "n_seq out of range");
  if (!page_tables || !start_pos || !n_ids) return fail(SR_E_INVALID, "null argument");
  if (m->tp_on() || m->d.tp_world > 1)
    return fail(SR_E_INVALID, "batched calls: tensor parallelism not supported");
  spans.resize(n_seq);
  int row = 0;
  for (int i = 0; i < n_seq; ++i) {
    if (!page_tables[i] || n_ids[i] < 1 || start_pos[i] < 0) return fail(SR_E_INVALID, "bad sequence");
    if (start_pos[i] + n_ids[i] > m->d.max_pos) return fail(SR_E_CAPACITY, "positions exceed max_pos");
    spans[i] = Model::SeqSpan{page_tables[i], start_pos[i], row, n_ids[i]};
    row += n_ids[i];
  }
  if (row > m->d.max_tokens) return fail(SR_E_CAPACITY, "batched rows exceed max_tokens");
  *total = row;
  return 0;
}

// run the pass, then the LM head over each sequence's last row (gathered into
// x rows 0..n_seq-1): fp32 logit partials in m->part [splits][n_seq][V]
static int batch_forward_last(Model* m, const std::vector<Model::SeqSpan>& spans, int M,
                              const int32_t* ids, const int32_t* tok_meta, cudaStream_t s) {
  const int n_seq = (int)spans.size();
  if ((size_t)n_seq * m->d.vocab_rows > m->L.part_floats)
    return fail(SR_E_CAPACITY, "LM-head partials exceed the workspace");
  if (int rc = m->run_layers(ids, M, spans.data(), n_seq, tok_meta, s)) return -rc;
  const size_t row_bytes = (size_t)m->d.d_model * sizeof(__nv_bfloat16);
  for (int i = 0; i < n_seq; ++i) {  // rows only move down: no copy overwrites a later source
    const int src = spans[i].row0 + spans[i].M - 1;
    if (src != i)
      SR_CK(cudaMemcpyAsync(m->x + (size_t)i * m->d.d_model, m->x + (size_t)src * m->d.d_model,
                            row_bytes, cudaMemcpyDeviceToDevice, s));
  }
  const int rc = m->gemm(Model::ACT_X, m->d.n_layers * 4, m->x, m->lm_head, n_seq,
                         m->d.vocab_rows, m->d.d_model, s);
  return rc ? -rc : 0;
}

int sr_score_batch(void* model, int32_t n_seq, const int32_t* const* page_tables,
                   const int32_t* start_pos, const int32_t* n_ids, const int32_t* ids,
                   const int32_t* tok_meta, const int8_t* first_digit, int32_t threshold,
                   sr_readout* readouts, void* stream) {
  Model* m = (Model*)model;
  if (!m || !ids || !tok_meta || !first_digit || !readouts) return fail(SR_E_INVALID, "null argument");
  std::vector<Model::SeqSpan> spans;
  int M = 0;
  if (int rc = batch_spans(m, n_seq, page_tables, start_pos, n_ids, spans, &M)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  SR_CK(cudaEventRecord(m->ev[0], s));
  if (int rc = batch_forward_last(m, spans, M, ids, tok_meta, s)) return rc;
  const size_t V = m->d.vocab_rows;
  for (int i = 0; i < n_seq; ++i) {
    ReadoutParams r{};
    if (m->last_splits == 1) {
      r.logits = m->part + (size_t)i * V;
    } else {
      SR_CK(split_sum_launch(m->part + (size_t)i * V, m->last_splits, (size_t)n_seq * V, m->logits,
                             V, s));
      r.logits = m->logits;
    }
    r.n_valid = m->d.vocab_text;
    r.first_digit = first_digit;
    r.threshold = threshold;
    r.counts = m->ro_cnt;
    r.part_v1 = m->lm_v1;
    r.part_v2 = m->lm_v2;
    r.part_i1 = m->lm_i1;
    r.out = readouts + i;
    SR_CK(readout_launch(r, m->num_sms, s));
  }
  SR_CK(cudaEventRecord(m->ev[1], s));
  SR_CK(cudaEventRecord(m->ev[2], s));
  m->timing.prefill_tokens = M;
  m->timing.decode_tokens = 0;
  return 0;
}

int sr_step_batch(void* model, int32_t n_seq, const int32_t* const* page_tables,
                  const int32_t* start_pos, const int32_t* n_ids, const int32_t* ids,
                  const int32_t* tok_meta, int32_t* out_ids, float* margins, void* stream) {
  Model* m = (Model*)model;
  if (!m || !ids || !tok_meta || !out_ids) return fail(SR_E_INVALID, "null argument");
  std::vector<Model::SeqSpan> spans;
  int M = 0;
  if (int rc = batch_spans(m, n_seq, page_tables, start_pos, n_ids, spans, &M)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  SR_CK(cudaEventRecord(m->ev[0], s));
  if (int rc = batch_forward_last(m, spans, M, ids, tok_meta, s)) return rc;
  const size_t V = m->d.vocab_rows;
  SR_CK(rows_argmax_launch(m->part, m->last_splits, (size_t)n_seq * V, n_seq, (int)V,
                           m->d.vocab_text, m->d.vocab_base, out_ids, margins, s, m->lm_v1,
                           m->lm_v2, m->lm_i1, m->lm_ctr, gemv_max_grid(m->num_sms) + 64));
  SR_CK(cudaEventRecord(m->ev[1], s));
  SR_CK(cudaEventRecord(m->ev[2], s));
  m->timing.prefill_tokens = M;
  m->timing.decode_tokens = 0;
  return 0;
}

int sr_tp_unique_id(uint8_t* h_id128) {
  if (!h_id128) return fail(SR_E_INVALID, "null argument");
  if (!tp_available()) return fail(SR_E_TP, "libnccl.so.2 not loadable");
  const int r = tp_unique_id(h_id128);
  return r ? fail(SR_E_TP, std::string("ncclGetUniqueId: ") + tp_error_string(r)) : 0;
}

int sr_tp_comm_create(const uint8_t* h_id128, int32_t world, int32_t rank, void** out_comm) {
  if (!h_id128 || !out_comm || world < 1 || world > 64 || rank < 0 || rank >= world)
    return fail(SR_E_INVALID, "bad communicator arguments");
  if (!tp_available()) return fail(SR_E_TP, "libnccl.so.2 not loadable");
  const int r = tp_comm_create(h_id128, world, rank, out_comm);
  return r ? fail(SR_E_TP, std::string("ncclCommInitRank: ") + tp_error_string(r)) : 0;
}

int sr_tp_comm_destroy(void* comm) {
  const int r = tp_comm_destroy(comm);
  return r ? fail(SR_E_TP, std::string("ncclCommDestroy: ") + tp_error_string(r)) : 0;
}

int sr_model_set_tp(void* model, void* comm) {
  Model* m = (Model*)model;
  if (!m) return fail(SR_E_INVALID, "null model");
  if (m->d.tp_world > 1 && !comm) return fail(SR_E_INVALID, "tp_world > 1 needs a communicator");
  m->tp_comm = comm;
  return 0;
}

// ----------------------------------------------- peer-memory TP transport ---
int sr_tp_peer_create(int32_t world, int32_t rank, int64_t max_elems, int32_t dec_row,
                      void** out_peer) {
  if (!out_peer || world < 1 || world > kPeerMaxWorld || rank < 0 || rank >= world ||
      max_elems < 16 || dec_row < 1)
    return fail(SR_E_INVALID, "bad peer transport arguments");
  PeerComm* pc = new PeerComm{};
  pc->world = world;
  pc->rank = rank;
  pc->max_elems = (size_t)max_elems;
  pc->dec_row = (dec_row + 63) / 64 * 64;
  peer_layout(pc);
  cudaError_t e = cudaMalloc((void**)&pc->local, pc->bytes);
  if (e == cudaSuccess) e = cudaMemset(pc->local, 0, pc->bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (pc->local) cudaFree(pc->local);
    delete pc;
    return fail(e, std::string("peer buffer: ") + cudaGetErrorString(e));
  }
  pc->base[rank] = pc->local;
  *out_peer = pc;
  return 0;
}

int sr_tp_peer_handle(void* peer, uint8_t* h_handle64) {
  PeerComm* pc = (PeerComm*)peer;
  if (!pc || !h_handle64) return fail(SR_E_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  SR_CK(cudaIpcGetMemHandle(&h, pc->local));
  memcpy(h_handle64, &h, sizeof(h));
  return 0;
}

int sr_tp_peer_open(void* peer, const uint8_t* h_handles) {
  PeerComm* pc = (PeerComm*)peer;
  if (!pc || !h_handles) return fail(SR_E_INVALID, "null argument");
  for (int q = 0; q < pc->world; ++q) {
    if (q == pc->rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, h_handles + (size_t)q * sizeof(h), sizeof(h));
    void* ptr = nullptr;
    SR_CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    pc->base[q] = (char*)ptr;
    pc->opened[q] = true;
  }
  return 0;
}

int sr_tp_peer_base(void* peer, uint64_t* h_base) {
  PeerComm* pc = (PeerComm*)peer;
  if (!pc || !h_base) return fail(SR_E_INVALID, "null argument");
  *h_base = (uint64_t)(uintptr_t)pc->local;
  return 0;
}

int sr_tp_peer_attach(void* peer, const uint64_t* h_bases) {
  PeerComm* pc = (PeerComm*)peer;
  if (!pc || !h_bases) return fail(SR_E_INVALID, "null argument");
  for (int q = 0; q < pc->world; ++q) {
    if (q == pc->rank) continue;
    if (!h_bases[q]) return fail(SR_E_INVALID, "null peer buffer");
    pc->base[q] = (char*)(uintptr_t)h_bases[q];
  }
  return 0;
}

int sr_tp_peer_destroy(void* peer) {
  PeerComm* pc = (PeerComm*)peer;
  if (!pc) return 0;
  for (int q = 0; q < pc->world; ++q)
    if (pc->opened[q]) cudaIpcCloseMemHandle(pc->base[q]);
  if (pc->local) cudaFree(pc->local);
  delete pc;
  return 0;
}

int sr_model_set_tp_peer(void* model, void* peer) {
  Model* m = (Model*)model;
  if (!m) return fail(SR_E_INVALID, "null model");
  PeerComm* pc = (PeerComm*)peer;
  if (!pc) {
    if (m->d.tp_world > 1 && !m->tp_comm) return fail(SR_E_INVALID, "tp_world > 1 needs a transport");
    m->tp_peer = nullptr;
    m->mk.tp_world = 1;
    return 0;
  }
  if (pc->world != m->d.tp_world || pc->rank != m->d.tp_rank)
    return fail(SR_E_INVALID, "peer transport world / rank differ from the model's");
  if (pc->dec_row < m->d.d_model || pc->max_elems < (size_t)m->d.max_tokens * m->d.d_model)
    return fail(SR_E_CAPACITY, "peer transport mailboxes smaller than the model needs");
  for (int q = 0; q < pc->world; ++q)
    if (!pc->base[q]) return fail(SR_E_INVALID, "peer transport not connected (open / attach)");
  m->tp_peer = pc;
  MkParams& p = m->mk;
  p.tp_world = pc->world;
  p.tp_rank = pc->rank;
  p.vocab_base = m->d.vocab_base;
  p.tp_dec_row = pc->dec_row;
  for (int q = 0; q < kPeerMaxWorld; ++q) p.tp_base[q] = q < pc->world ? pc->base[q] : nullptr;
  p.tp_off_dec = pc->off_dec;
  p.tp_off_lm = pc->off_lm;
  return 0;
}

int sr_model_set_decode_tiles(void* model, const uint64_t* h_ptrs) {
  Model* m = (Model*)model;
  if (!m) return fail(SR_E_INVALID, "null model");
  if (!h_ptrs) {
    m->mk.tiled = 0;
    return 0;
  }
  const int n = m->d.n_layers * 4 + 1;
  for (int i = 0; i < n; ++i)
    if (!h_ptrs[i] || (h_ptrs[i] & 15)) return fail(SR_E_INVALID, "tile-major weight pointer null or not 16-B aligned");
  // every tile's column count must be a multiple of 64 (the [32][64] boxes)
  const int K[4] = {m->d.d_model, m->q_dim, m->d.d_model, m->d.d_ffn};
  for (int i = 0; i < 4; ++i) {
    const int tc = std::min(K[i], mk_tile_cols());
    if (tc % 64 || K[i] % tc) return fail(SR_E_INVALID, "tile-major decode needs K % 64 == 0 and K % tile == 0");
  }
  SR_CK(cudaMemcpy(m->ws + m->L.mk_tiles, h_ptrs, n * sizeof(uint64_t), cudaMemcpyHostToDevice));
  m->mk.tiles = reinterpret_cast<const void* const*>(m->ws + m->L.mk_tiles);
  m->mk.tiled = 1;
  if (const char* v = getenv("SR_MK_TILED")) m->mk.tiled = atoi(v) != 0;
  return 0;
}

int sr_debug_profile(void* model, uint64_t* h_out, int32_t n) {
  Model* m = (Model*)model;
  if (!m || !h_out || n < 0) return fail(SR_E_INVALID, "null argument");
  if (n > SR_PROF_EVENTS) n = SR_PROF_EVENTS;
  SR_CK(cudaDeviceSynchronize());
  SR_CK(cudaMemcpy(h_out, m->ws + m->L.mk_prof, (size_t)n * 8, cudaMemcpyDeviceToHost));
  return 0;
}

int sr_debug_trace(void* model, int32_t* h_out, int32_t n) {
  Model* m = (Model*)model;
  if (!m || !h_out || !m->trace_host) return fail(SR_E_INVALID, "tracing is off (SR_MK_TRACE=1)");
  const int cap = m->num_sms * 8;
  for (int i = 0; i < n && i < cap; ++i) h_out[i] = ((volatile int*)m->trace_host)[i];
  return 0;
}

int sr_last_timing(void* model, sr_timing* h_out) {
  Model* m = (Model*)model;
  if (!m || !h_out) return fail(SR_E_INVALID, "null argument");
  float a = 0.f, b = 0.f;
  SR_CK(cudaEventSynchronize(m->ev[2]));
  SR_CK(cudaEventElapsedTime(&a, m->ev[0], m->ev[1]));
  SR_CK(cudaEventElapsedTime(&b, m->ev[1], m->ev[2]));
  m->timing.prefill_ms = a;
  m->timing.decode_ms = b;
  *h_out = m->timing;
  return 0;
}

}  // extern "C"
