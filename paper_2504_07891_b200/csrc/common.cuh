// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/specreason_b200.h"

#define SR_DEV __device__ __forceinline__

namespace sr {

constexpr int kHeadDim = SR_HEAD_DIM;
constexpr int kPage = SR_PAGE;
constexpr int kHalf = kHeadDim / 2;

// ---------------------------------------------------------------- PDL ------
// Programmatic dependent launch: a kernel may start while its predecessor
// drains; everything before grid_wait() must not read predecessor outputs.
SR_DEV void grid_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SR_DEV void grid_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------ loads -------
SR_DEV uint4 ld_stream(const void* p) {  // weights: read once, skip L1
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

SR_DEV void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

SR_DEV float2 bf2_to_f2(uint32_t v) {
  float2 r;
  r.x = __uint_as_float(v << 16);
  r.y = __uint_as_float(v & 0xffff0000u);
  return r;
}

SR_DEV float bf_to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

SR_DEV uint32_t f2_to_bf2(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}

SR_DEV float round_bf16(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// dot of 8 bf16 weights with 8 bf16 activations, fp32 accumulate
SR_DEV float dot8(uint4 w, uint4 x, float acc) {
  float2 a, b;
  a = bf2_to_f2(w.x); b = bf2_to_f2(x.x); acc = fmaf(a.x, b.x, acc); acc = fmaf(a.y, b.y, acc);
  a = bf2_to_f2(w.y); b = bf2_to_f2(x.y); acc = fmaf(a.x, b.x, acc); acc = fmaf(a.y, b.y, acc);
  a = bf2_to_f2(w.z); b = bf2_to_f2(x.z); acc = fmaf(a.x, b.x, acc); acc = fmaf(a.y, b.y, acc);
  a = bf2_to_f2(w.w); b = bf2_to_f2(x.w); acc = fmaf(a.x, b.x, acc); acc = fmaf(a.y, b.y, acc);
  return acc;
}

// ----------------------------------------------------------- reductions ---
SR_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

SR_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// block-wide sum; `red` must hold >= 32 floats; all threads get the result
SR_DEV float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float t = lane < nw ? red[lane] : 0.f;
  return warp_sum(t);
}

// (value, index) top-2 tracker: ties keep the lower index
struct Top2 {
  float v1, v2;
  int i1;
  SR_DEV void init() { v1 = -INFINITY; v2 = -INFINITY; i1 = 0x7fffffff; }
  SR_DEV void push(float v, int i) {
    if (v > v1 || (v == v1 && i < i1)) { v2 = v1; v1 = v; i1 = i; }
    else if (v > v2) v2 = v;
  }
  SR_DEV void merge(float ov1, int oi1, float ov2) {
    if (ov1 > v1 || (ov1 == v1 && oi1 < i1)) { v2 = fmaxf(v1, ov2); v1 = ov1; i1 = oi1; }
    else v2 = fmaxf(v2, ov1);
  }
};

SR_DEV void warp_top2(Top2& t) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov1 = __shfl_xor_sync(0xffffffffu, t.v1, o);
    float ov2 = __shfl_xor_sync(0xffffffffu, t.v2, o);
    int oi1 = __shfl_xor_sync(0xffffffffu, t.i1, o);
    t.merge(ov1, oi1, ov2);
  }
}

// --------------------------------------------- system-scope flag helpers ---
// (peer-memory collectives, tp.cu / decode_mk.cu): arrivals are release adds
// on a rank's flag word, waits acquire-poll the local flag
SR_DEV unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

SR_DEV void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

SR_DEV void peer_wait(const unsigned* flag, unsigned target) {
  const long long t0 = clock64();
  for (unsigned spin = 0;; ++spin) {
    if ((int)(ld_acquire_sys(flag) - target) >= 0) return;
    if ((spin & 4095) == 4095 && clock64() - t0 > 20000000000ll) __trap();  // ~10 s: a peer died
  }
}

// ------------------------------------------------------- layout helpers ---
// K/V pool: [layer][page][kv_head][SR_PAGE][128] bf16
SR_DEV size_t kv_offset(int layer, int page, int kvh, int slot, int n_pages, int n_kv) {
  return ((((size_t)layer * n_pages + page) * n_kv + kvh) * kPage + slot) * kHeadDim;
}

// ---------------------------------------------------------- decode state ---
// Lives in the workspace; kernels of a captured decode graph read it, so one
// graph serves every stream and position.
struct DecodeState {
  int pos;          // position of `token` (the token being fed)
  int token;        // token fed at `pos`
  int n_gen;        // tokens produced so far in this call
  int done;         // 1 once a stop / end-think / max_new is reached
  int finish;       // SR_FINISH_*
  int max_new;
  int ctx_len;      // pos + 1: K/V length the attention reads
  unsigned bar;     // grid-barrier counter of the persistent decode kernel (reset per call)
  const int* page_table;
  const uint8_t* token_class;
  int* out_ids;     // caller's out + 2
  int* out_hdr;     // caller's out (n_gen, finish)
  float* margins;   // may be null
  unsigned long long cond_handle;  // cudaGraphConditionalHandle of the while loop
  int pad1[2];
};

}  // namespace sr
