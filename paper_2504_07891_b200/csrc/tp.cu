#include <cstdio>
#include <cstdlib>
// Tensor parallelism of the base model.
//
// Megatron-style: each rank holds its q/k/v heads and gate/up units (column
// parallel) and the matching columns of O and down (row parallel); O and down
// therefore produce partial residual updates that are summed over ranks with
// an NCCL all-reduce over NVLink before the residual add.  The LM head is
// vocab-parallel: a greedy choice is the merge of every rank's (top-1, index,
// top-2), exchanged with one 12-byte-per-rank all-gather; the judge readout
// all-reduces ten digit rank counts.  The embedding and the norms are
// replicated.  NCCL is loaded with dlopen only when a communicator is created,
// so single-GPU users do not depend on it.
#include <dlfcn.h>

#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace sr {

// ------------------------------------------------------------ NCCL shim ---
namespace nccl {
typedef void* Comm;
struct UniqueId { char internal[128]; };
enum { kSum = 0, kInt32 = 2, kFloat32 = 7 };
typedef int (*GetUniqueIdFn)(UniqueId*);
typedef int (*CommInitRankFn)(Comm*, int, UniqueId, int);
typedef int (*CommDestroyFn)(Comm);
typedef int (*AllReduceFn)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*AllGatherFn)(const void*, void*, size_t, int, Comm, cudaStream_t);
typedef int (*BroadcastFn)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef const char* (*ErrStrFn)(int);

struct Api {
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  AllReduceFn all_reduce = nullptr;
  AllGatherFn all_gather = nullptr;
  BroadcastFn broadcast = nullptr;
  ErrStrFn err = nullptr;
  bool ok = false;
};

static Api& api() {
  static Api a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      a.get_unique_id = (GetUniqueIdFn)dlsym(h, "ncclGetUniqueId");
      a.comm_init_rank = (CommInitRankFn)dlsym(h, "ncclCommInitRank");
      a.comm_destroy = (CommDestroyFn)dlsym(h, "ncclCommDestroy");
      a.all_reduce = (AllReduceFn)dlsym(h, "ncclAllReduce");
      a.all_gather = (AllGatherFn)dlsym(h, "ncclAllGather");
      a.broadcast = (BroadcastFn)dlsym(h, "ncclBroadcast");
      a.err = (ErrStrFn)dlsym(h, "ncclGetErrorString");
      a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce &&
             a.all_gather && a.broadcast && a.err;
    }
  }
  return a;
}
}  // namespace nccl

int tp_available() { return nccl::api().ok ? 1 : 0; }
const char* tp_error_string(int code) {
  return nccl::api().ok ? nccl::api().err(code) : "libnccl.so.2 not loadable";
}

int tp_unique_id(void* out128) {
  if (!nccl::api().ok) return -1;
  nccl::UniqueId id;
  const int r = nccl::api().get_unique_id(&id);
  if (r == 0) memcpy(out128, id.internal, 128);
  return r;
}

int tp_comm_create(const void* id128, int world, int rank, void** out) {
  if (!nccl::api().ok) return -1;
  nccl::UniqueId id;
  memcpy(id.internal, id128, 128);
  nccl::Comm c = nullptr;
  const int r = nccl::api().comm_init_rank(&c, world, id, rank);
  if (r == 0) *out = c;
  return r;
}

int tp_comm_destroy(void* comm) { return comm ? nccl::api().comm_destroy(comm) : 0; }

int tp_all_reduce_f32(void* comm, float* buf, size_t n, cudaStream_t s) {
  return nccl::api().all_reduce(buf, buf, n, nccl::kFloat32, nccl::kSum, comm, s);
}
int tp_all_reduce_i32(void* comm, int* buf, size_t n, cudaStream_t s) {
  return nccl::api().all_reduce(buf, buf, n, nccl::kInt32, nccl::kSum, comm, s);
}
int tp_all_gather_f32(void* comm, const float* send, float* recv, size_t n, cudaStream_t s) {
  return nccl::api().all_gather(send, recv, n, nccl::kFloat32, comm, s);
}
int tp_broadcast_f32(void* comm, const float* send, float* recv, size_t n, int root,
                     cudaStream_t s) {
  return nccl::api().broadcast(send, recv, n, nccl::kFloat32, root, comm, s);
}

// ---------------------------------------------------------------- kernels ---
// delta[m][n] = sum of the split-K partials (fixed order)
__global__ void split_sum_kernel(const float* part, int splits, size_t stride, float* delta,
                                 size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    for (int s = 0; s < splits; ++s) v += __ldcg(part + s * stride + i);
    delta[i] = v;
  }
}

cudaError_t split_sum_launch(const float* part, int splits, size_t stride, float* delta, size_t n,
                             cudaStream_t s) {
  const int grid = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  split_sum_kernel<<<grid, 256, 0, s>>>(part, splits, stride, delta, n);
  return cudaGetLastError();
}

// h += delta; delta = 0   (decode: the all-reduced row-parallel output)
__global__ void add_delta_kernel(float* h, float* delta, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    h[i] += delta[i];
    delta[i] = 0.f;
  }
}

cudaError_t add_delta_launch(float* h, float* delta, int n, cudaStream_t s) {
  add_delta_kernel<<<(n + 255) / 256, 256, 0, s>>>(h, delta, n);
  return cudaGetLastError();
}

// local (top-1, top-2, global index) over this rank's logits -> send[3];
// the last CTA reduces the per-CTA partials (no extra launch)
__global__ void tp_top2_local_kernel(const float* logits, int n_valid, int base, float* pv1,
                                     float* pv2, int* pi1, unsigned* counter, float* send) {
  __shared__ float s1[8], s2[8];
  __shared__ int si[8];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Top2 b;
  b.init();
  for (int v = blockIdx.x * blockDim.x + tid; v < n_valid; v += gridDim.x * blockDim.x)
    b.push(logits[v], base + v);
  warp_top2(b);
  if (lane == 0) { s1[warp] = b.v1; s2[warp] = b.v2; si[warp] = b.i1; }
  __syncthreads();
  if (tid == 0) {
    Top2 c;
    c.init();
    for (int w = 0; w < 8; ++w) c.merge(s1[w], si[w], s2[w]);
    pv1[blockIdx.x] = c.v1;
    pv2[blockIdx.x] = c.v2;
    pi1[blockIdx.x] = c.i1;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  Top2 c;
  c.init();
  for (int i = tid; i < (int)gridDim.x; i += blockDim.x)
    c.merge(__ldcg(pv1 + i), __ldcg(pi1 + i), __ldcg(pv2 + i));
  warp_top2(c);
  if (lane == 0) { s1[warp] = c.v1; s2[warp] = c.v2; si[warp] = c.i1; }
  __syncthreads();
  if (tid == 0) {
    Top2 f;
    f.init();
    for (int w = 0; w < 8; ++w) f.merge(s1[w], si[w], s2[w]);
    send[0] = f.v1;
    send[1] = f.v2;
    send[2] = __int_as_float(f.i1);
    *counter = 0u;
  }
}

cudaError_t tp_top2_local_launch(const float* logits, int n_valid, int base, float* pv1,
                                 float* pv2, int* pi1, unsigned* counter, float* send, int grid,
                                 cudaStream_t s) {
  tp_top2_local_kernel<<<grid, 256, 0, s>>>(logits, n_valid, base, pv1, pv2, pi1, counter, send);
  return cudaGetLastError();
}

// merge the gathered [world][3] partials and take the greedy step
__global__ void tp_select_kernel(const float* gathered, int world, DecodeState* st) {
  Top2 f;
  f.init();
  for (int r = 0; r < world; ++r)
    f.merge(gathered[3 * r], __float_as_int(gathered[3 * r + 2]), gathered[3 * r + 1]);
  if (st->done) return;
  select_token(st, f.i1, f.v1 - f.v2);
}

cudaError_t tp_select_launch(const float* gathered, int world, DecodeState* st, cudaStream_t s) {
  tp_select_kernel<<<1, 1, 0, s>>>(gathered, world, st);
  return cudaGetLastError();
}

// judge readout, local pass: counts[d] = #{local valid v : logit_v > dig_d,
// or == with global id < d}; plus the local top-2 (send[10..12])
__global__ void tp_readout_local_kernel(const float* logits, int n_valid, int base,
                                        const float* dig, int* counts, float* pv1, float* pv2,
                                        int* pi1, unsigned* counter, float* send) {
  __shared__ unsigned cnt[10];
  __shared__ float s1[8], s2[8];
  __shared__ int si[8];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 10) cnt[tid] = 0;
  __syncthreads();
  float dl[10];
#pragma unroll
  for (int d = 0; d < 10; ++d) dl[d] = dig[d];
  unsigned c[10];
#pragma unroll
  for (int d = 0; d < 10; ++d) c[d] = 0;
  Top2 b;
  b.init();
  for (int v = blockIdx.x * blockDim.x + tid; v < n_valid; v += gridDim.x * blockDim.x) {
    const float x = logits[v];
    const int gv = base + v;
    b.push(x, gv);
#pragma unroll
    for (int d = 0; d < 10; ++d) c[d] += (x > dl[d] || (x == dl[d] && gv < d)) ? 1u : 0u;
  }
#pragma unroll
  for (int d = 0; d < 10; ++d) {
    unsigned t = c[d];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0 && t) atomicAdd(&cnt[d], t);
  }
  warp_top2(b);
  if (lane == 0) { s1[warp] = b.v1; s2[warp] = b.v2; si[warp] = b.i1; }
  __syncthreads();
  if (tid < 10 && cnt[tid]) atomicAdd(&counts[tid], (int)cnt[tid]);
  if (tid == 0) {
    Top2 f;
    f.init();
    for (int w = 0; w < 8; ++w) f.merge(s1[w], si[w], s2[w]);
    pv1[blockIdx.x] = f.v1;
    pv2[blockIdx.x] = f.v2;
    pi1[blockIdx.x] = f.i1;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  Top2 f;
  f.init();
  for (int i = tid; i < (int)gridDim.x; i += blockDim.x)
    f.merge(__ldcg(pv1 + i), __ldcg(pi1 + i), __ldcg(pv2 + i));
  warp_top2(f);
  if (lane == 0) { s1[warp] = f.v1; s2[warp] = f.v2; si[warp] = f.i1; }
  __syncthreads();
  if (tid == 0) {
    Top2 g;
    g.init();
    for (int w = 0; w < 8; ++w) g.merge(s1[w], si[w], s2[w]);
    send[0] = g.v1;
    send[1] = g.v2;
    send[2] = __int_as_float(g.i1);
    *counter = 0u;
  }
}

cudaError_t tp_readout_local_launch(const float* logits, int n_valid, int base, const float* dig,
                                    int* counts, float* pv1, float* pv2, int* pi1,
                                    unsigned* counter, float* send, int grid, cudaStream_t s) {
  tp_readout_local_kernel<<<grid, 256, 0, s>>>(logits, n_valid, base, dig, counts, pv1, pv2, pi1,
                                               counter, send);
  return cudaGetLastError();
}

// final readout from the all-reduced counts and the gathered top-2s; the
// preference order of extract_score (base.py:114-126)
__global__ void tp_readout_final_kernel(const float* dig, int* counts, const float* gathered,
                                        int world, const int8_t* first_digit, int threshold,
                                        sr_readout* out) {
  Top2 f;
  f.init();
  for (int r = 0; r < world; ++r)
    f.merge(gathered[3 * r], __float_as_int(gathered[3 * r + 2]), gathered[3 * r + 1]);
  int best = -1;
  float bv = -INFINITY, second = -INFINITY;
  for (int d = 0; d < 10; ++d) {
    if (counts[d] < 10) {
      if (best < 0 || dig[d] > bv) {
        second = best < 0 ? second : fmaxf(second, bv);
        best = d;
        bv = dig[d];
      } else {
        second = fmaxf(second, dig[d]);
      }
    }
  }
  int score = best;
  if (score < 0) score = first_digit[f.i1];
  sr_readout r;
  r.score = score;
  r.accept = (score >= 0 && score >= threshold) ? 1 : 0;
  r.margin = best >= 0 ? bv - second : 0.f;
  r.argmax = f.i1;
  *out = r;
  for (int d = 0; d < 10; ++d) counts[d] = 0;
}

cudaError_t tp_readout_final_launch(const float* dig, int* counts, const float* gathered,
                                    int world, const int8_t* first_digit, int threshold,
                                    sr_readout* out, cudaStream_t s) {
  tp_readout_final_kernel<<<1, 1, 0, s>>>(dig, counts, gathered, world, first_digit, threshold,
                                          out);
  return cudaGetLastError();
}

// ------------------------------------------------------- peer transport ---
// NVLink peer-memory collectives, no NCCL: every rank owns one exchange
// buffer (cudaMalloc, shared with the other ranks by CUDA IPC handles or, for
// ranks of one process, by plain device pointers).  A collective is one-shot:
// each rank stores its contribution into slot [rank] of every rank's mailbox
// (P2P stores over NVLink), then release-adds every rank's arrival flag; a
// rank reads only its own buffer, after acquiring its flag.  Sums run over
// ranks in rank order, so every rank computes bit-identical results.  Two
// mailbox slots alternate per channel: a rank writes slot s of exchange e+2
// only after exchange e+1 completed everywhere, i.e. after every rank read
// slot s of exchange e.
//
// Channels (flag words at the head of the buffer): host-driven collectives
// (prefill deltas, the first token's choice, judge readout) on flags 0-1;
// the persistent decode kernel's residual exchanges on flags 2-3 and its
// greedy merge on flags 4-5 (decode_mk.cu); words 8-9 count the kernel's
// exchanges across launches.
constexpr int kPeerBlocks = 16;
constexpr int kPeerThreads = 512;

static size_t peer_align(size_t v) { return (v + 255) & ~size_t(255); }

void peer_layout(PeerComm* pc) {
  size_t o = 256;  // flags + counters
  pc->off_dec = o;
  o = peer_align(o + (size_t)2 * pc->world * pc->dec_row * 4);
  pc->off_lm = o;
  o = peer_align(o + (size_t)2 * pc->world * 4 * 4);
  pc->off_big = o;
  o = peer_align(o + (size_t)2 * pc->world * pc->max_elems * 4);
  pc->bytes = o;
}

struct PeerX {
  char* base[kPeerMaxWorld];
  int world, rank, mode, root, slot;
  size_t off, max_elems, n;
  unsigned target;
  const float* send;
  float* recv;
};

// mode 0: all-reduce sum (f32), 1: all-gather (f32), 2: broadcast from root,
// 3: all-reduce sum (i32 bits)
__global__ void __launch_bounds__(kPeerThreads) peer_exchange_kernel(const PeerX x) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t slot_off = x.off + ((size_t)x.slot * x.world) * x.max_elems * 4;
  if (x.mode != 2 || x.rank == x.root) {
    for (size_t i = i0; i < x.n; i += stride) {
      const float v = x.send[i];
      for (int q = 0; q < x.world; ++q)
        reinterpret_cast<float*>(x.base[q] + slot_off)[(size_t)x.rank * x.max_elems + i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int q = 0; q < x.world; ++q)
      red_release_sys(reinterpret_cast<unsigned*>(x.base[q]) + x.slot, 1u);
    peer_wait(reinterpret_cast<const unsigned*>(x.base[x.rank]) + x.slot, x.target);
  }
  __syncthreads();
  const float* mb = reinterpret_cast<const float*>(x.base[x.rank] + slot_off);
  for (size_t i = i0; i < x.n; i += stride) {
    if (x.mode == 0) {
      float v = 0.f;
      for (int q = 0; q < x.world; ++q) v += __ldcg(mb + (size_t)q * x.max_elems + i);
      x.recv[i] = v;
    } else if (x.mode == 1) {
      for (int q = 0; q < x.world; ++q) x.recv[(size_t)q * x.n + i] = __ldcg(mb + (size_t)q * x.max_elems + i);
    } else if (x.mode == 2) {
      x.recv[i] = __ldcg(mb + (size_t)x.root * x.max_elems + i);
    } else {
      int v = 0;
      for (int q = 0; q < x.world; ++q) v += __float_as_int(__ldcg(mb + (size_t)q * x.max_elems + i));
      x.recv[i] = __int_as_float(v);
    }
  }
}

int peer_exchange(PeerComm* pc, int mode, const float* send, float* recv, size_t n, int root,
                  cudaStream_t s) {
  if (n > pc->max_elems) return -2;
  PeerX x{};
  for (int q = 0; q < pc->world; ++q) x.base[q] = pc->base[q];
  x.world = pc->world;
  x.rank = pc->rank;
  x.mode = mode;
  x.root = root;
  x.slot = (int)(pc->seq & 1u);
  x.off = pc->off_big;
  x.max_elems = pc->max_elems;
  x.n = n;
  // every block of every rank adds one to each flag per exchange
  x.target = (pc->seq / 2 + 1) * (unsigned)(pc->world * kPeerBlocks);
  x.send = send;
  x.recv = recv;
  pc->seq += 1;
  static const bool log = getenv("SR_TP_LOG") != nullptr;
  if (log) fprintf(stderr, "[peer] rank %d seq %u mode %d n %zu slot %d target %u\n", x.rank,
                   pc->seq - 1, mode, n, x.slot, x.target);
  peer_exchange_kernel<<<kPeerBlocks, kPeerThreads, 0, s>>>(x);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace sr
