// Kernel parameter blocks and host launchers shared by the runtime.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace sr {

// ------------------------------------------------------------------ GEMV ---
enum GemvKind {
  GEMV_QKV_EMBED,   // embed gather + RMSNorm -> qkv + bias + RoPE + K/V append
  GEMV_QKV,         // RMSNorm(h) -> qkv + bias + RoPE + K/V append
  GEMV_RESID,       // x -> h += W x
  GEMV_GLU,         // RMSNorm(h) -> silu(gate) * up
  GEMV_LM_ARGMAX,   // RMSNorm(h) -> logits -> greedy token (+ stop test)
  GEMV_LM_ARGMAX_X, // normalised x -> logits -> greedy token
  GEMV_LM_LOGITS_X, // normalised x -> fp32 logits
  GEMV_LM_LOGITS,   // RMSNorm(h) -> fp32 logits (vocab-parallel decode)
};

struct GemvParams {
  const __nv_bfloat16* W;
  int N, K, n_tasks, n_valid;
  const __nv_bfloat16* x;
  float* h;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* norm_w;
  float eps;
  // qkv epilogue
  const __nv_bfloat16* bias;
  const float* rope;
  __nv_bfloat16* qout;
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  int layer, n_pages, n_kv, q_dim, kv_dim;
  // glu / logits epilogues
  __nv_bfloat16* act_out;
  float* logits;
  // argmax epilogue
  float* part_v1;
  float* part_v2;
  int* part_i1;
  unsigned int* counter;
  int prefetch;  // issue L2 prefetches of the first task before the dependency wait
  DecodeState* st;
};

cudaError_t gemv_launch(GemvKind kind, GemvParams p, int num_sms, cudaStream_t stream, bool pdl);
int gemv_max_grid(int num_sms);

// Greedy choice bookkeeping + stop test, run by one thread (host mirror:
// paper_2504_07891_b200.host.finish_of).
SR_DEV void select_token(DecodeState* st, int t, float margin) {
  const int n = st->n_gen;
  st->out_ids[n] = t;
  if (st->margins) st->margins[n] = margin;
  const int cls = st->token_class[t];
  int done = 0, finish = SR_FINISH_LENGTH;
  if (cls == SR_CLASS_END_THINK) {
    done = 1;
    finish = SR_FINISH_END_THINK;
  } else if (cls == SR_CLASS_STOP) {
    done = 1;
    finish = SR_FINISH_STOP;
  } else if (n + 1 >= st->max_new) {
    done = 1;
  }
  st->n_gen = n + 1;
  st->done = done;
  st->finish = finish;
  if (!done) {
    st->token = t;
    st->pos = st->pos + 1;
    st->ctx_len = st->pos + 1;
  }
  st->out_hdr[0] = n + 1;
  st->out_hdr[1] = finish;
  if (st->cond_handle)
    cudaGraphSetConditional((cudaGraphConditionalHandle)st->cond_handle, done ? 0u : 1u);
}

// ------------------------------------------------------------- attention ---
struct AttnParams {
  const __nv_bfloat16* q;    // [M, H*128] (decode: M = 1)
  __nv_bfloat16* out;        // [M, H*128]
  const __nv_bfloat16* k_pool;
  const __nv_bfloat16* v_pool;
  const int* page_table;     // prefill; decode reads st->page_table
  float* part;               // [M, H, nsplit, 128 + 2]
  unsigned int* counters;    // [M, KV]
  int layer, n_pages, n_heads, n_kv, nsplit;
  int start_pos;             // prefill: position of row 0
  DecodeState* st;           // decode: ctx_len / page table from here
  // multi-sequence prefill (umma kernel): per grid-z item (first token, tokens,
  // start position, query tile of the span) and that span's page table
  const int4* spans;
  const int* const* span_tables;
};

int attn_decode_splits(int n_kv, int num_sms);
// tensor-core flash attention (attention_tc.cu)
cudaError_t attn_decode_tc_launch(const AttnParams& p, cudaStream_t stream, bool pdl);
cudaError_t attn_merge_launch(const AttnParams& p, int M_tokens, int nsplit, cudaStream_t stream);
// tcgen05 flash attention (attention_umma.cu); tmK / tmV: 128-B swizzled tensor
// maps over the K / V pools viewed as [rows = L*n_pages*n_kv*64, 128], box 64x64
cudaError_t attn_umma_launch(const void* tmK, const void* tmV, const AttnParams& p, int M_tokens,
                             int nsplit, cudaStream_t stream, int n_items = 0);
int attn_umma_splits(int n_kv, int q_tiles, int T, int num_sms);
int attn_umma_q_tiles(int M_tokens, int G);

// ----------------------------------------------------------- prefill path ---

// tcgen05 / TMEM / TMA version (gemm_tc.cu); tensor maps are CUtensorMap
// (128 B, 64-B aligned) built by make_tmap_bf16
struct TcGemmArgs {
  const void* tmW;  // W [N, K], box 64 x 128
  const void* tmX;  // X [M_cap, K], box 64 x tc_token_tile(M)
  float* C;         // [splits, M, N]
  int M, N, K, splits;
  __nv_bfloat16* act;  // non-null (splits == 1, interleaved gate/up W): write
                       // bf16 silu(gate) * up [M, N/2] instead of C
  int nt;              // token tile (0: tc_token_tile(M))
};
int tc_pick_tile(int M, int N, int num_sms);
int make_tmap_bf16(void* out_map, const void* ptr, int rows, int cols, int box_rows);
int make_tmap_bf16_box(void* out_map, const void* ptr, int rows, int cols, int box_cols,
                       int box_rows, bool swizzle128);
int tc_token_tile(int M);
int tc_pick_splits(int M, int N, int K, int num_sms, int nt = 0);
cudaError_t gemm_tc_launch(const TcGemmArgs& a, cudaStream_t stream);

struct EpiParams {
  const float* part;   // [splits, M, N]
  int splits, M, N;
  // residual + norm
  float* h;            // [M, d]
  const __nv_bfloat16* norm_w;
  float eps;
  __nv_bfloat16* x;    // [M, d] normalised output
  // qkv
  const __nv_bfloat16* bias;
  const float* rope;
  __nv_bfloat16* q;    // [M, q_dim]
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  const int* page_table;
  int start_pos, layer, n_pages, n_kv, q_dim, kv_dim;
  const int* tok_meta;  // multi-sequence passes: (position, page) per row; null:
                        // one sequence, position start_pos + row, page_table
  // glu
  __nv_bfloat16* act;  // [M, f]
};

cudaError_t embed_norm_launch(const int* ids, int M, const __nv_bfloat16* embed, int d,
                              const __nv_bfloat16* norm_w, float eps, float* h,
                              __nv_bfloat16* x, cudaStream_t stream);
cudaError_t epi_qkv_launch(const EpiParams& p, cudaStream_t stream);
cudaError_t epi_resid_norm_launch(const EpiParams& p, cudaStream_t stream);
cudaError_t epi_glu_launch(const EpiParams& p, cudaStream_t stream);

// per-row greedy choice over split LM-head partials (token-level speculation)
// (rows <= 16 with scratch: each row split over 16 CTAs; cv1/cv2/ci1 hold
// rows*16 chunk results, ctr one zeroed counter per row)
cudaError_t rows_argmax_launch(const float* part, int splits, size_t stride, int rows, int N,
                               int n_valid, int base, int32_t* out_ids, float* margins,
                               cudaStream_t stream, float* cv1 = nullptr, float* cv2 = nullptr,
                               int* ci1 = nullptr, unsigned* ctr = nullptr, int scratch = 0);

// verify readout over fp32 logits [V]
struct ReadoutParams {
  const float* logits;
  int n_valid;
  const int8_t* first_digit;
  int threshold;
  unsigned int* counts;  // [10] + [1] block counter
  float* part_v1;
  float* part_v2;
  int* part_i1;
  sr_readout* out;
};
cudaError_t readout_launch(const ReadoutParams& p, int num_sms, cudaStream_t stream);

// persistent weight-streaming decode kernel (decode_mk.cu)
#define SR_PROF_EVENTS 2048
struct MkLayer {
  const __nv_bfloat16* ln1;
  const __nv_bfloat16* bqkv;
  const __nv_bfloat16* ln2;
  const void* pad;
};

constexpr int kPeerMaxWorld = 8;  // ranks of a peer-memory TP group

struct MkParams {
  const CUtensorMap* maps;   // device [L*4 + 1]: per layer qkv, o, gate/up, down; then LM head
  const MkLayer* layers;     // device [L]
  const __nv_bfloat16* embed;
  const __nv_bfloat16* ln_f;
  const float* rope;
  __nv_bfloat16* k_pool;
  __nv_bfloat16* v_pool;
  float* hA;                 // residual stream, two alternating buffers [d]
  float* hB;
  const uint16_t* ctab;      // [3][256] per 32-row block of qkv / o / down: first CTA |
                             // #contributors << 8 | slot << 12 (host-built)
  int* attn_cnt;             // [KV] split tickets of the attention merge
  float* part_qkv;           // [G][maxj][32] split-row partials
  float* part_o;
  float* part_d;
  float* apart;              // [G][8][130] attention split partials
  float* lm_part;            // [G][3] per-CTA (top1, top2, index)
  __nv_bfloat16* act;        // [f]
  __nv_bfloat16* attn;       // [q_dim]
  DecodeState* st;
  volatile int* trace;       // SR_MK_TRACE: mapped host [G][8] progress words, or null
  unsigned long long* prof;  // SR_MK_PROF: [SR_PROF_EVENTS] globaltimer stamps, or null
  int L, d, H, KV, f, vocab_rows, vocab_text, n_pages, q_dim, kv_dim, qkv_rows;
  float eps;
  int maxj, stages, xs_elems;
  int l2_ahead;              // tiles prefetched into L2 beyond the shared-memory ring
  int head_split;            // split a page's query heads over idle CTAs (short contexts)
  int combine_wide;          // COMBINE items of 64 dims (1), 32 dims (0), or by item count (-1)
  int bar_sleep;             // ns of backoff between grid-barrier polls
  int evict_first;           // stream weights with an L2 evict-first policy
  int min_pages;             // attention: minimum K/V pages per split
  int kv_dbl;                // attention pages double-buffered (second buffer in the x region)
  int vec_prologue;          // norm prologues: 16-B loads, one batch (SR_MK_VECPRO=0: scalar)
  // tile-major decode weights (sr_model_set_decode_tiles): per layer qkv, o,
  // gate/up, down, then the LM head; tile (b, k) of a matrix is 32 rows x tc
  // columns at ((b * kt) + k) * 32 * tc * 2 bytes, stored as tc / 64 boxes of
  // [32][64] with the 128-B swizzle applied; null = row-major + TMA 2-D boxes
  const void* const* tiles;
  int tiled;                 // 1: stream tiles by 1-D bulk copy, GEMV on mma.sync
  int no_load;               // SR_MK_NOLOAD experiment: stages handed out without loading
                             // weights (times the consumer chain alone; results invalid)
  // tensor parallelism over NVLink peer memory (tp_world > 1): every rank's
  // exchange buffer (flags at the head, tp.cu), the decode / greedy mailboxes
  int tp_world, tp_rank, vocab_base, tp_dec_row;
  char* tp_base[kPeerMaxWorld];
  size_t tp_off_dec, tp_off_lm;
};

size_t mk_smem_bytes(int stages, int xs_elems, int kv_dbl);
int mk_pick_stages(int xs_elems);
int mk_pick_kv_dbl(int stages, int xs_elems);
int mk_max_j(int N, int K, int num_sms);
int mk_tile_rows();
int mk_tile_cols();
cudaError_t mk_launch(const MkParams& p, int num_sms, cudaStream_t stream);

// NVLink peer-memory transport (tp.cu): one exchange buffer per rank
struct PeerComm {
  int world, rank;
  int dec_row;                       // floats per rank row of the decode mailbox (>= d_model)
  size_t max_elems;                  // floats per rank of the host-collective mailbox
  size_t off_dec, off_lm, off_big, bytes;
  char* local;                       // this rank's buffer (cudaMalloc)
  char* base[kPeerMaxWorld];         // every rank's buffer in this device's address space
  bool opened[kPeerMaxWorld];        // opened through cudaIpcOpenMemHandle
  unsigned seq;                      // host-driven exchanges issued so far
};
void peer_layout(PeerComm* pc);
// mode 0: all-reduce sum f32, 1: all-gather f32 (recv [world][n]), 2: broadcast
// from root, 3: all-reduce sum i32; returns 0, or < 0 on a launch / size error
int peer_exchange(PeerComm* pc, int mode, const float* send, float* recv, size_t n, int root,
                  cudaStream_t s);

// tensor parallelism (tp.cu)
int tp_available();
const char* tp_error_string(int code);
int tp_unique_id(void* out128);
int tp_comm_create(const void* id128, int world, int rank, void** out);
int tp_comm_destroy(void* comm);
int tp_all_reduce_f32(void* comm, float* buf, size_t n, cudaStream_t s);
int tp_all_reduce_i32(void* comm, int* buf, size_t n, cudaStream_t s);
int tp_all_gather_f32(void* comm, const float* send, float* recv, size_t n, cudaStream_t s);
int tp_broadcast_f32(void* comm, const float* send, float* recv, size_t n, int root,
                     cudaStream_t s);
cudaError_t split_sum_launch(const float* part, int splits, size_t stride, float* delta, size_t n,
                             cudaStream_t s);
cudaError_t add_delta_launch(float* h, float* delta, int n, cudaStream_t s);
cudaError_t tp_top2_local_launch(const float* logits, int n_valid, int base, float* pv1,
                                 float* pv2, int* pi1, unsigned* counter, float* send, int grid,
                                 cudaStream_t s);
cudaError_t tp_select_launch(const float* gathered, int world, DecodeState* st, cudaStream_t s);
cudaError_t tp_readout_local_launch(const float* logits, int n_valid, int base, const float* dig,
                                    int* counts, float* pv1, float* pv2, int* pi1,
                                    unsigned* counter, float* send, int grid, cudaStream_t s);
cudaError_t tp_readout_final_launch(const float* dig, int* counts, const float* gathered,
                                    int world, const int8_t* first_digit, int threshold,
                                    sr_readout* out, cudaStream_t s);

// decode-loop bookkeeping kernels
cudaError_t decode_begin_launch(DecodeState* st, const DecodeState* h_init, cudaStream_t stream,
                                const int32_t* feed = nullptr);
cudaError_t cond_init_launch(DecodeState* st, unsigned long long handle, cudaStream_t stream);

}  // namespace sr
