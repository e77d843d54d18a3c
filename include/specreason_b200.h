/*
 * specreason_b200.h -- C-ABI of the B200-native SpecReason inner loop.
 *
 * The reference (arXiv 2504.07891, package `stepspec`) has no native code: its
 * only device crossing is the OpenAI-completions POST of the HTTP backend
 * (pkg/src/stepspec/backends/http.py:63-94) behind the `Backend` plugin API
 * (pkg/src/stepspec/backends/base.py:77-100).  This library replaces what sits
 * behind that POST -- the model server -- with sm_100a kernels; the Python
 * shim (paper_2504_07891_b200/backend.py) keeps the `Backend` API itself.
 *
 * Entry points and the reference interface each one replaces:
 *
 *   sr_generate  <- Backend.generate_step (base.py:87-89); semantics of
 *                   OpenAICompletionsBackend.generate_step (http.py:121-152):
 *                   prefill the fresh prompt suffix, greedy decode, stop at a
 *                   stop-class token (kept) or </think> (dropped), else at
 *                   max_new (finish "length").
 *   sr_score     <- Backend.score_step (base.py:91-97); semantics of
 *                   OpenAICompletionsBackend.score_step (http.py:154-174) +
 *                   extract_score (base.py:106-126) + decide_acceptance
 *                   (core.py:91-93): one prefill pass, digit readout over the
 *                   top-10 of the last position, threshold compare.  Only the
 *                   16-byte sr_readout leaves the GPU.
 *   page tables  <- _PrefixLedger streams (engine.py:161-186): the caller owns
 *                   page allocation; truncating a stream (rollback) is just a
 *                   shorter start_pos on the next call; prefilling the suffix
 *                   is the commit.
 *
 * Ownership: the caller (PyTorch on the Python side) allocates every buffer --
 * weights, K/V page pools, workspace, outputs.  The library never allocates
 * device memory for data; it keeps only CUDA graphs and kernel attributes in
 * the opaque sr_model handle.  All pointers are device pointers unless named
 * h_*; `stream` is a cudaStream_t passed as void*.
 *
 * Errors: every int-returning call returns 0 on success, else a cudaError_t
 * value or one of SR_E_*; sr_last_error() returns the thread-local message.
 * Calls on one sr_model must be serialised by the caller (one stream at a
 * time); distinct models are independent.
 */
#ifndef SPECREASON_B200_H
#define SPECREASON_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SR_ABI_VERSION 1
#define SR_PAGE 64            /* tokens per K/V page */
#define SR_HEAD_DIM 128

#define SR_E_INVALID 1001     /* bad descriptor / argument */
#define SR_E_CAPACITY 1002    /* request exceeds a compiled or declared limit */
#define SR_E_GRAPH 1003       /* CUDA graph construction failed */
#define SR_E_TP 1004          /* NCCL unavailable or a collective failed */

/* finish codes written to sr_generate's output */
#define SR_FINISH_LENGTH 0
#define SR_FINISH_STOP 1
#define SR_FINISH_END_THINK 2

/* token classes of the per-request class table (uint8 per LM-head row) */
#define SR_CLASS_PLAIN 0
#define SR_CLASS_STOP 1
#define SR_CLASS_END_THINK 2
#define SR_CLASS_MASKED 3

typedef struct sr_model_desc {
  int32_t n_layers;
  int32_t d_model;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t head_dim;     /* must be SR_HEAD_DIM */
  int32_t d_ffn;
  int32_t vocab_rows;   /* embedding / LM-head rows */
  int32_t vocab_text;   /* rows >= vocab_text are never produced */
  float rms_eps;
  int32_t max_pos;      /* rows of the RoPE table; positions must be < max_pos */
  int32_t max_tokens;   /* largest n_ids of one prefill call */
  int32_t max_new;      /* largest max_new of one sr_generate call */
  int32_t n_pages;      /* pages in each of the K and V pools */
  /* tensor parallelism (1 = off).  The caller passes this rank's shard
   * (heads, ffn units and LM-head rows divided by tp_world; embedding and
   * norms whole) and attaches a communicator with sr_model_set_tp. */
  int32_t tp_world;
  int32_t tp_rank;
  int32_t vocab_base;   /* global token id of LM-head row 0 of this shard */
} sr_model_desc;

typedef struct sr_layer_ptrs {
  const void* ln1;   /* bf16 [d] */
  const void* wqkv;  /* bf16 [(H + 2*KV)*128, d]: q rows, k rows, v rows */
  const void* bqkv;  /* bf16 [(H + 2*KV)*128] */
  const void* wo;    /* bf16 [d, H*128] */
  const void* ln2;   /* bf16 [d] */
  const void* wgu;   /* bf16 [2*f, d]: gate/up interleaved in 16-row blocks */
  const void* wd;    /* bf16 [d, f] */
} sr_layer_ptrs;

typedef struct sr_model_ptrs {
  const void* embed;          /* bf16 [vocab_rows, d] */
  const void* ln_f;           /* bf16 [d] */
  const void* lm_head;        /* bf16 [vocab_rows, d] */
  const sr_layer_ptrs* layers;/* host array [n_layers] */
  const float* rope;          /* fp32 [max_pos, 64, 2] (cos, sin) */
  void* k_pool;               /* bf16 [n_layers, n_pages, KV, SR_PAGE, 128] */
  void* v_pool;               /* same */
  void* workspace;            /* sr_workspace_bytes(desc) bytes, 256-B aligned */
} sr_model_ptrs;

typedef struct sr_readout {   /* 16 bytes, the only verify output */
  int32_t score;              /* 0..9, or -1 = no digit (ScoreParseFailure) */
  int32_t accept;             /* score >= threshold (0 when score == -1) */
  float margin;               /* best digit logit - runner-up digit logit */
  int32_t argmax;             /* greedy token at the last position */
} sr_readout;

typedef struct sr_timing {    /* optional per-call device timings (ms) */
  float prefill_ms;
  float decode_ms;
  int32_t prefill_tokens;
  int32_t decode_tokens;
} sr_timing;

int sr_abi_version(void);
const char* sr_last_error(void);

/* bytes of workspace the caller must provide for `desc` */
size_t sr_workspace_bytes(const sr_model_desc* desc);

int sr_model_create(const sr_model_desc* desc, const sr_model_ptrs* ptrs, void* stream,
                    void** out_model);
int sr_model_destroy(void* model);

/*
 * Prefill ids[0..n_ids) at positions start_pos.. of the stream whose page
 * table is `page_table` (int32, one page id per SR_PAGE positions, covering
 * start_pos + n_ids + max_new positions), then greedy-decode up to max_new
 * tokens.  out (int32): out[0] = tokens generated, out[1] = finish code,
 * out[2 .. 2+max_new) = token ids; margins (fp32 [max_new], may be NULL) =
 * top-1 minus top-2 logit of each choice.  K/V of every fed token (prompt
 * suffix and all generated tokens but the last) is resident on return.
 */
int sr_generate(void* model, const int32_t* page_table, int32_t start_pos,
                const int32_t* ids, int32_t n_ids, int32_t max_new,
                const uint8_t* token_class, int32_t* out, float* margins,
                void* stream);

/*
 * Prefill ids at start_pos.. and read the judge digit at the last position:
 * rank_d = #{v : logit_v > logit_d, or == with v < d}; the best digit with
 * rank < 10 wins (lower id on ties); else the first digit character of the
 * greedy token's text (first_digit[v], int8, -1 = none); accept = score >=
 * threshold.  Writes one sr_readout to `readout` (device).
 */
int sr_score(void* model, const int32_t* page_table, int32_t start_pos,
             const int32_t* ids, int32_t n_ids, const int8_t* first_digit,
             int32_t threshold, sr_readout* readout, void* stream);

/*
 * Token-level speculation (SpecReason+Decode): prefill ids at start_pos..
 * (n_ids <= max_tokens) and write the greedy choice after every fed token:
 * out_ids[i] = argmax of the logits at position start_pos + i (ties: lower
 * id), margins[i] (may be NULL) = top-1 minus top-2.  The LM head runs as
 * one tensor-core GEMM over all rows.
 */
int sr_verify_tokens(void* model, const int32_t* page_table, int32_t start_pos,
                     const int32_t* ids, int32_t n_ids, int32_t* out_ids, float* margins,
                     void* stream);

/*
 * Multi-sequence passes (several trajectories per GPU).  n_seq
 * streams (n_seq <= 64) each feed n_ids[i] fresh tokens at positions
 * start_pos[i].. of their own page table page_tables[i] (host array of device
 * pointers; start_pos, n_ids: host arrays).  ids (device) holds the
 * sequences' tokens back to back, sum(n_ids) <= max_tokens; tok_meta (device,
 * int32 pairs) holds (position, page id) of every row.  One weight stream
 * serves all rows; attention runs per sequence.
 *
 * sr_score_batch: the judge readout of sr_score at each sequence's last row,
 *   readouts[i] (device).
 * sr_step_batch: the greedy choice at each sequence's last row, out_ids[i]
 *   (ties: lower id) and margins[i] (may be NULL) -- one batched decode step
 *   when every n_ids[i] == 1, the first token after a prompt otherwise.
 */
int sr_score_batch(void* model, int32_t n_seq, const int32_t* const* page_tables,
                   const int32_t* start_pos, const int32_t* n_ids, const int32_t* ids,
                   const int32_t* tok_meta, const int8_t* first_digit, int32_t threshold,
                   sr_readout* readouts, void* stream);
int sr_step_batch(void* model, int32_t n_seq, const int32_t* const* page_tables,
                  const int32_t* start_pos, const int32_t* n_ids, const int32_t* ids,
                  const int32_t* tok_meta, int32_t* out_ids, float* margins, void* stream);

/*
 * Test hook: prefill ids and write fp32 logits of every new position
 * (`all` != 0, logits [n_ids, vocab_rows]) or of the last one ([vocab_rows]).
 */
int sr_forward_logits(void* model, const int32_t* page_table, int32_t start_pos,
                      const int32_t* ids, int32_t n_ids, int32_t all, float* logits,
                      void* stream);

/*
 * Tensor parallelism over NCCL (loaded with dlopen on first use).  Rank 0
 * creates the 128-byte id, the caller distributes it, every rank creates its
 * communicator and attaches it to its model.  With a communicator attached,
 * O and down partial outputs are all-reduced (fp32 sum) before the residual
 * add, greedy choices merge an all-gathered (top-1, index, top-2) per rank,
 * and the judge readout all-reduces the ten digit rank counts.
 */
int sr_tp_unique_id(uint8_t* h_id128);
int sr_tp_comm_create(const uint8_t* h_id128, int32_t world, int32_t rank, void** out_comm);
int sr_tp_comm_destroy(void* comm);
int sr_model_set_tp(void* model, void* comm);

/*
 * Tensor parallelism over NVLink peer memory (no NCCL).  Each rank creates
 * one exchange buffer (sr_tp_peer_create: max_elems floats per rank for the
 * host-driven collectives -- at least max_tokens * d_model -- and dec_row >=
 * d_model floats per rank for the decode kernel's mailbox), shares it with
 * the other ranks (sr_tp_peer_handle / sr_tp_peer_open over CUDA IPC across
 * processes; sr_tp_peer_base / sr_tp_peer_attach within one process) and
 * attaches it to its model (sr_model_set_tp_peer).  With it the persistent
 * decode kernel decodes a tensor-parallel step itself: after the O and down
 * phases each CTA stores its rows of the rank's partial residual update into
 * every rank's mailbox and the ranks sum them in rank order; the greedy
 * choice merges every rank's (top-1, index, top-2).  Prefill and the judge
 * readout use one-shot peer all-reduce / all-gather / broadcast kernels, or
 * NCCL when a communicator is attached too.
 */
int sr_tp_peer_create(int32_t world, int32_t rank, int64_t max_elems, int32_t dec_row,
                      void** out_peer);
int sr_tp_peer_handle(void* peer, uint8_t* h_handle64);
int sr_tp_peer_open(void* peer, const uint8_t* h_handles);   /* world x 64 bytes, rank order */
int sr_tp_peer_base(void* peer, uint64_t* h_base);
int sr_tp_peer_attach(void* peer, const uint64_t* h_bases); /* world device pointers */
int sr_tp_peer_destroy(void* peer);
int sr_model_set_tp_peer(void* model, void* peer);

/*
 * Decode-layout weights (no reference counterpart: an HBM layout choice of
 * the persistent decode kernel).  h_ptrs: n_layers * 4 + 1 device pointers --
 * per layer qkv, o, gate/up, down, then the LM head -- each matrix [N][K]
 * re-stored tile-major: tile (b, k) = rows 32b..32b+31 x columns k*tc..
 * (tc = min(K, 256)), tiles in (b, k) order, each tile as tc/64 boxes of
 * [32 rows][64 columns] with the 128-B swizzle applied (16-B chunk j of row r
 * at r * 128 + ((j ^ (r & 7)) << 4)).  The decode kernel then streams each
 * 16 KB tile with one contiguous bulk copy and runs its GEMVs on mma.sync.
 * The row-major weights of sr_model_create stay in use for prefill.  NULL
 * detaches them (row-major TMA boxes, CUDA-core GEMV).
 */
int sr_model_set_decode_tiles(void* model, const uint64_t* h_ptrs);

/* device timings of the last sr_generate / sr_score on this model */
int sr_last_timing(void* model, sr_timing* h_out);

/*
 * Profiling hook: with SR_MK_PROF=1 in the environment at sr_model_create,
 * the persistent decode kernel records globaltimer stamps (ns) of CTA 0 after
 * every phase of the first decoded token of each sr_generate; copies the
 * first n (<= 2048) of them to h_out.
 */
int sr_debug_profile(void* model, uint64_t* h_out, int32_t n);

/*
 * Bring-up hook: with SR_MK_TRACE=1 at sr_model_create, every CTA of the
 * persistent decode kernel publishes progress words (step, stages consumed,
 * barrier target, stages issued, tokens) to mapped host memory [#SMs][8];
 * readable (no CUDA call) even while a kernel hangs.
 */
int sr_debug_trace(void* model, int32_t* h_out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* SPECREASON_B200_H */
