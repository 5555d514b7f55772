// Device-initiated exchange over NVLink peer memory (the B200-native K3/K4/K5).
//
// Replaces the modelled PS push/pull (sparseplan/simulate.py:183-240) and the
// server-side aggregation + update (simulate.py:294-323) without NCCL and
// without host synchronisation, so a whole multi-GPU step is CUDA-graph
// capturable:
//
//   worker: send rows (send order, dest-major)  --k_push-->  owner inboxes
//           (NVLink stores, then per-owner {count, epoch} flags)
//   owner : k_wait(push flags) -> k_owner_scatter (slot table, no sort)
//           -> k_owner_apply (sum in source order, optimizer, reset)
//           -> {epoch} "applied" flags to every peer
//   worker: k_wait(applied flags) -> k_pull (peer reads of the updated rows)
//
// Windows: each rank cudaMallocs one symmetric window per table and exports
// it with cudaIpc; peers map it. Layout (offsets from the window base):
//   [sig]   int32 push_flag[n], push_count[n], applied_flag[n], epoch, err
//   [w]     the rank's table slab [rows_cap, D] fp32 (peer-readable)
//   [ids]   inbox ids  [n][cap] int64   (source-major)
//   [rows]  inbox rows [n][cap][D] fp32
// Spin-waits run in ONE small block (k_wait) and give up after a bounded time,
// raising an error bit instead of hanging the GPU.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "hp_common.cuh"

namespace hp {
namespace {

constexpr int SIG_INTS = 4 * 64 + 64;  // up to 64 ranks

struct SigView {
  int* push_flag;     // [n] epoch of the last push received from source s
  int* push_count;    // [n] rows received from source s
  int* applied_flag;  // [n] epoch of the last apply finished by owner o
  int* epoch;         // [1] this rank's step epoch
  int* err;           // [1]
  int* done;          // [4] last-block counters
  __host__ __device__ explicit SigView(void* base) {
    int* b = static_cast<int*>(base);
    push_flag = b;
    push_count = b + 64;
    applied_flag = b + 128;
    epoch = b + 192;
    err = b + 193;
    done = b + 196;
  }
};

__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct PeerTable {
  void* base[64];  // window base of every rank (own rank = local pointer)
};

// ---- push: copy this rank's dest-major send blocks into the owners' inboxes.
// One warp per row; the last block to finish publishes {count, epoch}.
__global__ void __launch_bounds__(256)
k_push(PeerTable peers, int n, int me, int64_t w_off, int64_t ids_off, int64_t rows_off,
       int64_t cap, int D4, const int64_t* __restrict__ send_ids,
       const float4* __restrict__ send_rows, const int32_t* __restrict__ dest_counts,
       int total_bound, void* my_win) {
  __shared__ int s_off[65];
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    int run = 0;
    for (int o = 0; o < n; ++o) {
      s_off[o] = run;
      run += dest_counts[o];
    }
    s_off[n] = run;
  }
  __syncthreads();
  const int total = s_off[n];
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < total; k += nw) {
    int o = 0;
    while (o + 1 < n && k >= s_off[o + 1]) ++o;
    const int64_t slot = (int64_t)me * cap + (k - s_off[o]);
    char* win = static_cast<char*>(peers.base[o]);
    float4* dst = reinterpret_cast<float4*>(win + rows_off) + slot * D4;
    const float4* src = send_rows + (int64_t)k * D4;
    for (int c = lane; c < D4; c += 32) dst[c] = src[c];
    if (lane == 0) reinterpret_cast<int64_t*>(win + ids_off)[slot] = send_ids[k];
  }
  (void)total_bound;
  (void)w_off;
  // publish: every block fences its peer stores, the last one raises the flags
  __threadfence_system();
  __syncthreads();
  SigView me_sig(my_win);
  if (threadIdx.x == 0) s_last = atomicAdd(&me_sig.done[0], 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    const int e = *me_sig.epoch + 1;
    for (int o = threadIdx.x; o < n; o += blockDim.x) {
      SigView peer(peers.base[o]);
      peer.push_count[me] = s_off[o + 1] - s_off[o];
      __threadfence_system();
      st_release_sys(&peer.push_flag[me], e);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      *me_sig.epoch = e;
      me_sig.done[0] = 0;
    }
  }
}

// ---- wait until flags[s] >= epoch for every s (one block; bounded spin).
__global__ void k_wait(void* my_win, int which, int n, long long timeout_cycles) {
  SigView sig(my_win);
  const int* flags = which == 0 ? sig.push_flag : sig.applied_flag;
  const int e = *sig.epoch;
  for (int s = threadIdx.x; s < n; s += blockDim.x) {
    const long long t0 = clock64();
    while (ld_acquire_sys(&flags[s]) < e) {
      if (clock64() - t0 > timeout_cycles) {
        atomicOr(sig.err, which == 0 ? 4 : 8);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence();
}

// ---- owner: direct-mapped merge. slot[row * n + s] = inbox index of source s
// for slab row `row` (or -1); every row is listed once in `list`.
__global__ void __launch_bounds__(256)
k_owner_scatter(void* my_win, int n, int64_t ids_off, int64_t cap, const int64_t* __restrict__ part_base,
                Router route, int32_t* slot, int32_t* touch, int32_t* list, int32_t* nlist,
                int64_t rows_cap) {
  SigView sig(my_win);
  const int64_t* inbox_ids = reinterpret_cast<const int64_t*>(static_cast<char*>(my_win) + ids_off);
  const int64_t total = (int64_t)n * cap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / cap);
    const int k = (int)(i - (int64_t)s * cap);
    if (k >= sig.push_count[s]) continue;
    const int64_t id = inbox_ids[i];
    const int p = route.part(id);
    const int64_t b = part_base[p];
    const int64_t row = b + (id - route.lo(p));
    if (b < 0 || row >= rows_cap) {
      atomicOr(sig.err, 16);
      continue;
    }
    slot[row * n + s] = (int32_t)i;
    if (atomicAdd(&touch[row], 1) == 0) list[atomicAdd(nlist, 1)] = (int32_t)row;
  }
}

template <int OPT>
__device__ __forceinline__ void opt_update(float& w, float& a, float& b, float g, const hp_optim& o) {
  g = __fmul_rn(g, o.agg_scale);
  if (OPT == HP_OPT_SGD) {
    w = __fsub_rn(w, __fmul_rn(o.lr, g));
  } else if (OPT == HP_OPT_ADAGRAD) {
    a = __fadd_rn(a, __fmul_rn(g, g));
    w = __fsub_rn(w, __fdiv_rn(__fmul_rn(o.lr, g), __fsqrt_rn(a)));
  } else {
    a = __fadd_rn(__fmul_rn(o.beta1, a), __fmul_rn(o.one_minus_beta1, g));
    b = __fadd_rn(__fmul_rn(o.beta2, b), __fmul_rn(o.one_minus_beta2, __fmul_rn(g, g)));
    w = __fsub_rn(w, __fdiv_rn(__fmul_rn(o.lr_t, a), __fadd_rn(__fsqrt_rn(b), o.eps)));
  }
}

// ---- owner: per listed row, sum the (<= n) contributions in source order,
// scale, apply, reset the slot table; last block raises "applied" at peers.
template <int OPT>
__global__ void __launch_bounds__(256)
k_owner_apply(PeerTable peers, void* my_win, int n, int me, int64_t w_off, int64_t rows_off, int D4,
              float4* s0, float4* s1, hp_optim o, int32_t* slot, int32_t* touch,
              const int32_t* __restrict__ list, int32_t* nlist, int list_bound) {
  __shared__ bool s_last;
  SigView sig(my_win);
  char* win = static_cast<char*>(my_win);
  float4* w = reinterpret_cast<float4*>(win + w_off);
  const float4* inbox = reinterpret_cast<const float4*>(win + rows_off);
  const int nl = *nlist;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < nl; k += nw) {
    const int64_t row = list[k];
    int src[64];
    int ns = 0;
    for (int s = 0; s < n; ++s) {
      const int v = slot[row * n + s];
      if (v >= 0) src[ns++] = v;
    }
    for (int c = lane; c < D4; c += 32) {
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = 0; j < ns; ++j) g = f4_add(g, inbox[(int64_t)src[j] * D4 + c]);
      const int64_t off = row * D4 + c;
      float4 wv = w[off];
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (OPT != HP_OPT_SGD) a = s0[off];
      if (OPT == HP_OPT_ADAM) b = s1[off];
      opt_update<OPT>(wv.x, a.x, b.x, g.x, o);
      opt_update<OPT>(wv.y, a.y, b.y, g.y, o);
      opt_update<OPT>(wv.z, a.z, b.z, g.z, o);
      opt_update<OPT>(wv.w, a.w, b.w, g.w, o);
      w[off] = wv;
      if (OPT != HP_OPT_SGD) s0[off] = a;
      if (OPT == HP_OPT_ADAM) s1[off] = b;
    }
    __syncwarp();
    if (lane < n) slot[row * n + lane] = -1;
    if (lane == 0) touch[row] = 0;
  }
  (void)list_bound;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&sig.done[1], 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    const int e = *sig.epoch;
    for (int r = threadIdx.x; r < n; r += blockDim.x) st_release_sys(&SigView(peers.base[r]).applied_flag[me], e);
    if (threadIdx.x == 0) {
      sig.done[1] = 0;
      *nlist = 0;
    }
  }
}

// ---- worker pull: pulled[k] = updated row of send slot k, read from its owner.
__global__ void __launch_bounds__(256)
k_pull(PeerTable peers, int64_t w_off, int D4, const int64_t* __restrict__ send_ids,
       const int32_t* __restrict__ n_uniq, const int32_t* __restrict__ owner,
       const int64_t* __restrict__ glob_base, Router route, float4* pulled) {
  const int U = *n_uniq;
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < U; k += nw) {
    const int64_t id = send_ids[k];
    const int p = route.part(id);
    const float4* src = reinterpret_cast<const float4*>(static_cast<char*>(peers.base[owner[p]]) + w_off) +
                        (glob_base[p] + (id - route.lo(p))) * D4;
    for (int c = lane; c < D4; c += 32) pulled[(int64_t)k * D4 + c] = src[c];
  }
}

}  // namespace
}  // namespace hp

using namespace hp;

// Spin-wait budget (cycles) before a wait gives up and raises an error bit.
static long long wait_budget() {
  static long long v = [] {
    const char* e = getenv("HP_WAIT_TIMEOUT_CYCLES");
    return e ? atoll(e) : 4000000000LL;  // ~2 s at 1.9 GHz
  }();
  return v;
}

// Opaque exchange state for one table (declared in include/hybridpath.h).
struct hp_xchg_s {
  int n, me, D;
  int64_t cap, rows_cap;
  int64_t w_off, ids_off, rows_off, bytes;
  void* win;            // own window
  PeerTable peers;      // mapped windows (own = win)
  int32_t* slot;        // [rows_cap * n]
  int32_t* touch;       // [rows_cap]
  int32_t* list;        // [min(n*cap, rows_cap)]
  int32_t* nlist;       // [1]
};
extern "C" {

size_t hp_xchg_window_bytes(int32_t n, int32_t D, int64_t cap, int64_t rows_cap) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return al(SIG_INTS * 4) + al((size_t)rows_cap * D * 4) + al((size_t)n * cap * 8) +
         al((size_t)n * cap * D * 4);
}

int hp_xchg_create(hp_xchg_t* out, int32_t n, int32_t me, int32_t D, int64_t cap, int64_t rows_cap,
                   void* ipc_handle_out /* 64 bytes */, void** w_out) {
  HP_REQUIRE(out && ipc_handle_out && w_out && n >= 1 && n <= 64 && me >= 0 && me < n, "bad xchg args");
  HP_REQUIRE(D % 4 == 0 && D >= 4 && cap >= 1 && rows_cap >= 1, "bad xchg shape");
  auto* x = new hp_xchg_s{};
  x->n = n;
  x->me = me;
  x->D = D;
  x->cap = cap;
  x->rows_cap = rows_cap;
  auto al = [](int64_t v) { return (v + 255) & ~(int64_t)255; };
  x->w_off = al(SIG_INTS * 4);
  x->ids_off = x->w_off + al(rows_cap * D * 4);
  x->rows_off = x->ids_off + al((int64_t)n * cap * 8);
  x->bytes = x->rows_off + al((int64_t)n * cap * D * 4);
  cudaError_t e = cudaMalloc(&x->win, x->bytes);
  if (e != cudaSuccess) { delete x; return cuda_fail(e, "cudaMalloc(window)"); }
  HP_CUDA(cudaMemset(x->win, 0, SIG_INTS * 4));
  cudaIpcMemHandle_t h;
  HP_CUDA(cudaIpcGetMemHandle(&h, x->win));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(ipc_handle_out, &h, sizeof(h));
  const int64_t lb = std::min<int64_t>((int64_t)n * cap, rows_cap);
  HP_CUDA(cudaMalloc(&x->slot, (size_t)rows_cap * n * 4));
  HP_CUDA(cudaMemset(x->slot, 0xff, (size_t)rows_cap * n * 4));
  HP_CUDA(cudaMalloc(&x->touch, (size_t)rows_cap * 4));
  HP_CUDA(cudaMemset(x->touch, 0, (size_t)rows_cap * 4));
  HP_CUDA(cudaMalloc(&x->list, (size_t)std::max<int64_t>(lb, 1) * 4));
  HP_CUDA(cudaMalloc(&x->nlist, 4));
  HP_CUDA(cudaMemset(x->nlist, 0, 4));
  for (int r = 0; r < 64; ++r) x->peers.base[r] = nullptr;
  x->peers.base[me] = x->win;
  *w_out = static_cast<char*>(x->win) + x->w_off;
  *out = x;
  return HP_OK;
}

int hp_xchg_open_peer(hp_xchg_t x, int32_t rank, const void* ipc_handle) {
  HP_REQUIRE(x && rank >= 0 && rank < x->n && ipc_handle, "bad peer args");
  if (rank == x->me) return HP_OK;
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  void* p = nullptr;
  HP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  x->peers.base[rank] = p;
  return HP_OK;
}

int hp_xchg_destroy(hp_xchg_t x) {
  if (!x) return HP_OK;
  for (int r = 0; r < x->n; ++r)
    if (r != x->me && x->peers.base[r]) cudaIpcCloseMemHandle(x->peers.base[r]);
  cudaFree(x->slot);
  cudaFree(x->touch);
  cudaFree(x->list);
  cudaFree(x->nlist);
  cudaFree(x->win);
  delete x;
  return HP_OK;
}

// Push this rank's send blocks to the owners and raise the push flags.
int hp_xchg_push(hp_xchg_t x, const int64_t* send_ids, const float* send_rows,
                 const int32_t* dest_counts, int64_t T_bound, void* stream) {
  HP_REQUIRE(x && send_ids && send_rows && dest_counts, "NULL argument");
  HP_REQUIRE(T_bound <= x->cap, "more rows than the inbox capacity");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = grid_for(T_bound, 8, sm_count() * 4);
  k_push<<<blocks, 256, 0, st>>>(x->peers, x->n, x->me, x->w_off, x->ids_off, x->rows_off, x->cap,
                                 x->D / 4, send_ids, reinterpret_cast<const float4*>(send_rows),
                                 dest_counts, (int)T_bound, x->win);
  HP_LAUNCHED(1, "k_push");
  return HP_OK;
}

// Owner: wait for every source's push, merge + apply into the slab, signal peers.
int hp_xchg_merge_apply(hp_xchg_t x, hp_slab slab, hp_optim opt, void* stream) {
  HP_REQUIRE(x && slab.part_base, "NULL argument");
  HP_REQUIRE(slab.D == x->D, "slab width differs from the exchange");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_wait<<<1, 64, 0, st>>>(x->win, 0, x->n, wait_budget());
  const int64_t total = (int64_t)x->n * x->cap;
  k_owner_scatter<<<grid_for(total, 256, sm_count() * 8), 256, 0, st>>>(
      x->win, x->n, x->ids_off, x->cap, slab.part_base, Router(slab.V, slab.P), x->slot, x->touch,
      x->list, x->nlist, x->rows_cap);
  const int lb = (int)std::min<int64_t>(total, x->rows_cap);
  const int blocks = grid_for(lb, 8, sm_count() * 4);
  float4* s0 = reinterpret_cast<float4*>(slab.s0);
  float4* s1 = reinterpret_cast<float4*>(slab.s1);
  const int D4 = x->D / 4;
  switch (opt.kind) {
    case HP_OPT_SGD:
      k_owner_apply<HP_OPT_SGD><<<blocks, 256, 0, st>>>(x->peers, x->win, x->n, x->me, x->w_off,
                                                       x->rows_off, D4, s0, s1, opt, x->slot,
                                                       x->touch, x->list, x->nlist, lb);
      break;
    case HP_OPT_ADAGRAD:
      k_owner_apply<HP_OPT_ADAGRAD><<<blocks, 256, 0, st>>>(x->peers, x->win, x->n, x->me,
                                                           x->w_off, x->rows_off, D4, s0, s1, opt,
                                                           x->slot, x->touch, x->list, x->nlist, lb);
      break;
    default:
      k_owner_apply<HP_OPT_ADAM><<<blocks, 256, 0, st>>>(x->peers, x->win, x->n, x->me, x->w_off,
                                                        x->rows_off, D4, s0, s1, opt, x->slot,
                                                        x->touch, x->list, x->nlist, lb);
  }
  HP_LAUNCHED(3, "owner merge/apply");
  return HP_OK;
}

// Worker: wait for every owner's apply, then read the updated rows of its
// unique ids (send order) from the owners' slabs. glob_base[p] = slab row of
// partition p on its owner.
int hp_xchg_pull(hp_xchg_t x, const int64_t* send_ids, const int32_t* n_uniq, int64_t T_bound,
                 const int32_t* owner, const int64_t* glob_base, int64_t V, int32_t P,
                 float* pulled, void* stream) {
  HP_REQUIRE(x && send_ids && n_uniq && owner && glob_base && pulled, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_wait<<<1, 64, 0, st>>>(x->win, 1, x->n, wait_budget());
  k_pull<<<grid_for(T_bound, 8, sm_count() * 4), 256, 0, st>>>(
      x->peers, x->w_off, x->D / 4, send_ids, n_uniq, owner, glob_base, Router(V, P),
      reinterpret_cast<float4*>(pulled));
  HP_LAUNCHED(2, "pull");
  return HP_OK;
}

// Rows received from each source in the last push (device copy, stream-ordered).
// Debug: copy the window's signal words (push_flag[64], push_count[64],
// applied_flag[64], epoch, err, ...) to a host buffer of >= 200 ints (syncs).
int hp_xchg_debug_sig(hp_xchg_t x, int32_t* host_out, void* stream) {
  HP_REQUIRE(x && host_out, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_CUDA(cudaMemcpyAsync(host_out, x->win, 200 * 4, cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  return HP_OK;
}

int hp_xchg_recv_counts(hp_xchg_t x, int32_t* out_dev, void* stream) {
  HP_REQUIRE(x && out_dev, "NULL argument");
  SigView sig(x->win);
  HP_CUDA(cudaMemcpyAsync(out_dev, sig.push_count, 4 * (size_t)x->n, cudaMemcpyDeviceToDevice,
                          static_cast<cudaStream_t>(stream)));
  return HP_OK;
}

// Error bits of the exchange (4: push wait timed out, 8: apply wait timed out,
// 16: a received id is not homed here). Synchronises the stream.
int hp_xchg_status(hp_xchg_t x, int32_t* out_err, void* stream) {
  HP_REQUIRE(x && out_err, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SigView sig(x->win);
  HP_CUDA(cudaMemcpyAsync(out_err, sig.err, 4, cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  return HP_OK;
}

}  // extern "C"
