// Device-initiated exchange over NVLink peer memory (the B200-native K3/K4/K5).
//
// Replaces the modelled PS push/pull (sparseplan/simulate.py:183-240) and the
// server-side aggregation + update (simulate.py:294-323) without NCCL and
// without host synchronisation, so a whole multi-GPU step is CUDA-graph
// capturable. Compute and communication are fused:
//
//   worker  dedup plan (k_dedup_*), then k_reduce/k_combine with EpiPush: every
//           summed row is stored straight into its owner's inbox over NVLink,
//           and an epoch-tagged entry {epoch, inbox index} into the owner's
//           direct-mapped slot table [slab row][source]; the last k_combine
//           block publishes {count, offset, epoch} per owner.
//   owner   k_wait(push) -> k_owner_apply: one warp per inbox entry; the entry
//           of the lowest-ranked source of a row (valid tags) owns the row:
//           sums the contributions in source order, optimizer update, and
//           stores the updated row straight back into every contributor's
//           return buffer (NVLink); last block publishes "applied". No sort,
//           no atomics, no reset (stale tags never match the epoch).
//   worker  k_wait(applied) -> stitch from the local return buffer.
//
// Windows: each rank cudaMallocs one symmetric window per table and exports
// it with cudaIpc; peers map it. Layout (offsets from the window base):
//   [sig]   int32 push_flag[64], push_count[64], applied_flag[64], epoch, err,
//           done[4], push_off[64]
//   [w]     the rank's table slab [rows_cap, D] fp32 (peer-readable)
//   [ids]   inbox ids  [n][cap] int64   (source-major)
//   [rows]  inbox rows [n][cap][D] fp32
//   [ret]   return rows [cap][D] fp32 (indexed by this rank's send slot)
//   [slot]  uint64 [rows_cap][n] = (epoch << 32) | inbox index (peer-written)
// Spin-waits run in ONE small block (k_wait) and give up after a bounded time,
// raising an error bit instead of hanging the GPU.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cuda_bf16.h>

#include "hp_reduce.cuh"

namespace hp {
namespace {

constexpr int SIG_INTS = 5 * 64;  // up to 64 ranks

struct SigView {
  int* push_flag;     // [n] epoch of the last push received from source s
  int* push_count;    // [n] rows received from source s
  int* applied_flag;  // [n] epoch of the last apply finished by owner o
  int* epoch;         // [1] this rank's step epoch
  int* err;           // [1]
  int* done;          // [4] last-block counters
  int* push_off;      // [n] source s's send offset of its block for this owner
  int* own_items;     // [1] owner merge items written by k_owner_scan this step
  __host__ __device__ explicit SigView(void* base) {
    int* b = static_cast<int*>(base);
    push_flag = b;
    push_count = b + 64;
    applied_flag = b + 128;
    epoch = b + 192;
    err = b + 193;
    done = b + 196;
    push_off = b + 256;
    own_items = b + 194;
  }
};

// Fork / join events of the split push (hp_xchg_push_plan with a side
// stream), per device; recorded and waited on back to back, so two suffice.
cudaEvent_t push_event(int k) {
  static cudaEvent_t ev[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!ev[dev][k]) cudaEventCreateWithFlags(&ev[dev][k], cudaEventDisableTiming);
  return ev[dev][k];
}

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

struct WinLayout {
  int64_t w_off, ids_off, rows_off, ret_off, slot_off, items_off, cidx_off, cap;
  int n, me, D4;
};

// ---- push epilogue: the summed row of send slot `dst` goes to its owner's inbox.
// The destination of every send slot {inbox index, owner, slab row} was
// resolved on the plan stream (k_send_info), so load() issues independent
// loads only and the item's row loads are not held behind an index chain.
struct EpiPush {
  static constexpr bool kRemote = true;
  static constexpr bool kOut = false;
  static constexpr int kPre = 0;
  __device__ __forceinline__ const float4* pre_row(int, int) const { return nullptr; }
  PeerTable peers;
  WinLayout L;
  const int32_t* dest_counts;  // [n] rows this rank sends to each owner
  const int64_t* send_ids;     // [U] (send order)
  const int4* info;            // [U] {inbox index, owner, slab row, 0}
  void* my_win;
  struct Pre {
    int4 inf;
    int64_t id;
    int epoch;
  };
  __device__ __forceinline__ Pre load(int slot, int c4) const {
    Pre p;
    p.inf = info[slot];
    if (c4 == 0) {
      p.id = send_ids[slot];
      p.epoch = *SigView(my_win).epoch + 1;
    }
    return p;
  }
  __device__ __forceinline__ void store(int, int c4, float4 g, const Pre& p) const {
    char* win = static_cast<char*>(peers.base[p.inf.y]);
    reinterpret_cast<float4*>(win + L.rows_off)[(int64_t)p.inf.x * L.D4 + c4] = g;
    if (c4 == 0) {
      reinterpret_cast<int64_t*>(win + L.ids_off)[p.inf.x] = p.id;
      reinterpret_cast<unsigned long long*>(win + L.slot_off)[(int64_t)p.inf.z * L.n + L.me] =
          ((unsigned long long)(unsigned)p.epoch << 32) | (unsigned long long)(uint32_t)p.inf.x;
    }
  }
  // Runs once, in k_publish after k_combine (after a system fence that covers
  // every peer store of the reduce): publish {count, offset}, then the epoch
  // flag at every owner.
  __device__ void grid_done() const {
    SigView me(my_win);
    const int e = *me.epoch + 1;
    for (int o = threadIdx.x; o < L.n; o += blockDim.x) {
      int off = 0;
      for (int q = 0; q < o; ++q) off += dest_counts[q];
      SigView peer(peers.base[o]);
      peer.push_count[L.me] = dest_counts[o];
      peer.push_off[L.me] = off;
      st_release_sys(&peer.push_flag[L.me], e);  // release: orders this thread's stores above
    }
    __syncthreads();
    if (threadIdx.x == 0) *me.epoch = e;
  }
};

// ---- plan stream: destination of every send slot u < U (owners in ascending
// rank order, each owner's block of slots contiguous): inbox index
// me * cap + (u - first slot of the owner), owner rank, slab row at the owner.
__global__ void k_send_info(const int64_t* __restrict__ send_ids, const int32_t* __restrict__ dest_counts,
                            const int32_t* __restrict__ n_uniq, const int64_t* __restrict__ glob_base,
                            Router route, WinLayout L, int4* __restrict__ info, int64_t T) {
  const int U = *n_uniq;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U && u < T;
       u += (int64_t)gridDim.x * blockDim.x) {
    int o = 0, off = 0;
    while (o + 1 < L.n && u >= off + dest_counts[o]) off += dest_counts[o++];
    const int64_t id = send_ids[u];
    const int p = route.part(id);
    const int64_t row = glob_base[p] + (id - route.lo(p));
    info[u] = make_int4((int)((int64_t)L.me * L.cap + (u - off)), o, (int)row, 0);
  }
}

// ---- wait until flags[s] >= epoch - lag for every s (one block; bounded
// spin). lag > 0: an earlier bucket of a bucketed dense exchange.
__global__ void k_wait(void* my_win, int which, int n, long long timeout_cycles, int span, int lag) {
  HP_ENTRY(span);
  SigView sig(my_win);
  const int* flags = which == 0 ? sig.push_flag : sig.applied_flag;
  const int e = *sig.epoch - lag;
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
  HP_SPAN_END(span);
}

template <int OPT>
__device__ __forceinline__ void opt_update(float& w, float& a, float& b, float g,
                                           const hp_optim& o) {
  g = __fmul_rn(g, o.agg_scale);
  if (OPT == HP_OPT_SGD) {
    w = __fsub_rn(w, __fmul_rn(o.lr, g));
  } else if (OPT == HP_OPT_ADAGRAD) {
    a = __fadd_rn(a, __fmul_rn(g, g));
    w = __fsub_rn(w, __fdiv_rn(__fmul_rn(o.lr, g), __fsqrt_rn(a)));
  } else {
    a = __fadd_rn(__fmul_rn(o.beta1, a), __fmul_rn(o.one_minus_beta1, g));
    b = __fadd_rn(__fmul_rn(o.beta2, b), __fmul_rn(o.one_minus_beta2, __fmul_rn(g, g)));
    w = __fsub_rn(w, __fdiv_rn(__fmul_rn(adam_lr_t(o), a), __fadd_rn(__fsqrt_rn(b), o.eps)));
  }
}

// ---- owner: one group of TPI threads per inbox entry (source s, index k);
// each thread owns VPT float4 columns, so a row is one load round trip. The
// entry of the lowest-ranked source with a valid tag for its row owns the row:
// it sums the contributions in source order, scales, applies, and stores the
// updated row back into every contributor's return buffer (peer stores). The
// last block raises "applied".
template <int OPT, int TPI, int VPT>
__global__ void __launch_bounds__(256, VPT >= 4 ? 2 : 3)
k_owner_apply(PeerTable peers, void* my_win, WinLayout L, const int64_t* __restrict__ part_base,
              Router route, float4* s0, float4* s1, hp_optim o, int64_t rows_cap) {
  __shared__ bool s_last;
  HP_ENTRY(SP_APPLY);
  SigView sig(my_win);
  char* win = static_cast<char*>(my_win);
  float4* w = reinterpret_cast<float4*>(win + L.w_off);
  const float4* inbox = reinterpret_cast<const float4*>(win + L.rows_off);
  const int64_t* inbox_ids = reinterpret_cast<const int64_t*>(win + L.ids_off);
  const unsigned long long* slot = reinterpret_cast<const unsigned long long*>(win + L.slot_off);
  const int n = L.n, D4 = L.D4;
  const unsigned epoch = (unsigned)*sig.epoch;
  const int lane = threadIdx.x & 31, q = threadIdx.x % TPI;
  constexpr int GPB = 256 / TPI;
  // after a push wait timed out (error bit 4) nothing is merged (see k_owner_scan)
  const int64_t total =
      (*reinterpret_cast<volatile int*>(sig.err) & 4) ? 0 : (int64_t)n * L.cap;
  for (int64_t e = (int64_t)blockIdx.x * GPB + threadIdx.x / TPI; e < total;
       e += (int64_t)gridDim.x * GPB) {
    const int s = (int)(e / L.cap);
    if (e - (int64_t)s * L.cap >= sig.push_count[s]) continue;  // group-uniform
    const int64_t id = inbox_ids[e];
    const int p = route.part(id);
    const int64_t b = part_base[p];
    const int64_t row = b + (id - route.lo(p));
    if (b < 0 || row >= rows_cap) {
      if (q == 0) atomicOr(sig.err, 16);
      continue;
    }
    const unsigned long long ent = lane < n ? slot[row * n + lane] : 0ull;
    const bool valid = lane < n && (unsigned)(ent >> 32) == epoch;
    const unsigned have = __ballot_sync(0xffffffffu, valid);
    if (__ffs(have) - 1 != s) continue;  // another source's entry owns this row
    const int cnt = __popc(have);
    const int from = lane < cnt ? (int)__fns(have, 0, lane + 1) : lane;
    const int cidx = __shfl_sync(0xffffffffu, (int)(uint32_t)ent, from);
    float4 wv[VPT], av[VPT], bv[VPT], g[VPT];
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c = q + v * TPI;
      const int64_t off = row * D4 + c;
      wv[v] = av[v] = bv[v] = g[v] = z;
      if (c < D4) {
        wv[v] = w[off];
        if (OPT != HP_OPT_SGD) av[v] = s0[off];
        if (OPT == HP_OPT_ADAM) bv[v] = s1[off];
      }
    }
    for (int j0 = 0; j0 < cnt; j0 += 2) {  // contributions, in source order
      float4 x[2][VPT];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = __shfl_sync(0xffffffffu, cidx, (j0 + u) & 31);
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (j0 + u < cnt && q + v * TPI < D4) x[u][v] = inbox[(int64_t)idx * D4 + q + v * TPI];
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (j0 + u < cnt) g[v] = f4_add(g[v], x[u][v]);
    }
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c = q + v * TPI;
      if (c >= D4) continue;
      opt_update<OPT>(wv[v].x, av[v].x, bv[v].x, g[v].x, o);
      opt_update<OPT>(wv[v].y, av[v].y, bv[v].y, g[v].y, o);
      opt_update<OPT>(wv[v].z, av[v].z, bv[v].z, g[v].z, o);
      opt_update<OPT>(wv[v].w, av[v].w, bv[v].w, g[v].w, o);
      const int64_t off = row * D4 + c;
      w[off] = wv[v];
      if (OPT != HP_OPT_SGD) s0[off] = av[v];
      if (OPT == HP_OPT_ADAM) s1[off] = bv[v];
    }
    // pull, fused: the updated row goes back to each contributor's send slot
    for (int j = 0; j < cnt; ++j) {
      const int idx = __shfl_sync(0xffffffffu, cidx, j);
      const int src = idx / (int)L.cap;
      const int64_t ret_row = sig.push_off[src] + (idx - (int64_t)src * L.cap);
      float4* ret = reinterpret_cast<float4*>(static_cast<char*>(peers.base[src]) + L.ret_off) +
                    ret_row * D4;
#pragma unroll
      for (int v = 0; v < VPT; ++v)
        if (q + v * TPI < D4) ret[q + v * TPI] = wv[v];
    }
  }
  // one cumulative system-scope release per block (after the barrier) orders
  // every thread's peer stores before the block's arrival
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_last = atomicAdd(&sig.done[1], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      st_release_sys(&SigView(peers.base[r]).applied_flag[L.me], (int)epoch);
    if (threadIdx.x == 0) sig.done[1] = 0;
  }
  HP_SPAN_END(SP_APPLY);
}

// ---- owner, streamed: the same merge/apply as k_owner_apply, restructured
// as a per-warp row stream (k_rowstream's pipeline). Warp w takes a contiguous
// range of the valid inbox entries (all sources, source-major). Per batch of
// 32 entries the lanes load ids and slot-table tags in parallel (two
// coalesced/independent round trips per 32 entries instead of two per entry)
// and decide ownership; then every owned entry becomes cnt contribution rows
// (source order) followed by the optimizer's state rows, copied global ->
// shared with cp.async, F = S - kPre rows in flight per warp. The END element
// applies the update from shared memory, stores w/state locally and the new
// row into each contributor's return buffer over NVLink.
constexpr int OS_NMAX = HP_CHUNK;  // contributors per row (n <= HP_CHUNK)

struct OsMeta {
  int64_t row;
  int flags, cnt;
  int cidx[OS_NMAX];
};

template <int OPT, int VPT, int S>
__global__ void __launch_bounds__(128)
k_owner_stream(PeerTable peers, void* my_win, WinLayout L, const int64_t* __restrict__ part_base,
               Router route, float4* s0, float4* s1, hp_optim o, int64_t rows_cap) {
  constexpr int D4 = VPT * 32;
  constexpr int KPRE = OPT == HP_OPT_SGD ? 1 : (OPT == HP_OPT_ADAGRAD ? 2 : 3);
  constexpr int F = S - KPRE;
  static_assert(F >= 2, "owner stream needs >= 2 rows in flight");
  extern __shared__ __align__(16) float4 s_rows[];  // [4][S][D4]
  __shared__ OsMeta s_meta[4][S];
  __shared__ int s_cid[4][32][OS_NMAX];  // contributor list of the current batch, per lane
  __shared__ int s_pre[OS_NMAX + 1];     // prefix of valid entries per source
  __shared__ int s_poff[OS_NMAX];
  __shared__ bool s_last;
  HP_ENTRY(SP_APPLY);
  SigView sig(my_win);
  char* win = static_cast<char*>(my_win);
  float4* w = reinterpret_cast<float4*>(win + L.w_off);
  const float4* inbox = reinterpret_cast<const float4*>(win + L.rows_off);
  const int64_t* inbox_ids = reinterpret_cast<const int64_t*>(win + L.ids_off);
  const unsigned long long* slot = reinterpret_cast<const unsigned long long*>(win + L.slot_off);
  const int n = L.n;
  const unsigned epoch = (unsigned)*sig.epoch;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    int a = 0;
    for (int q = 0; q < n; ++q) {
      s_pre[q] = a;
      a += sig.push_count[q];
      s_poff[q] = sig.push_off[q];
    }
    s_pre[n] = a;
  }
  __syncthreads();
  const int E = (*reinterpret_cast<volatile int*>(sig.err) & 4) ? 0 : s_pre[n];
  const int NW = gridDim.x * 4, gw = blockIdx.x * 4 + wid;
  const int Q = (E + NW - 1) / NW;
  const int fb0 = min(E, gw * Q), fe = min(E, fb0 + Q);
  float4* ring = s_rows + (size_t)wid * S * D4;
  const float4* pre_base[3] = {w, s0, s1};

  // batch state (lane l <-> entry fb + l)
  int fb = fb0;
  unsigned own_mask = 0;
  int64_t my_row = 0;
  int my_cnt = 0;
  auto load_batch = [&]() {
    const int f = fb + lane;
    bool owned = false;
    my_cnt = 0;
    if (f < fe) {
      int sidx = 0;
      while (sidx + 1 < n && f >= s_pre[sidx + 1]) ++sidx;
      const int64_t e = (int64_t)sidx * L.cap + (f - s_pre[sidx]);
      const int64_t id = inbox_ids[e];
      const int p = route.part(id);
      const int64_t b = part_base[p];
      const int64_t row = b + (id - route.lo(p));
      if (b < 0 || row >= rows_cap) {
        atomicOr(sig.err, 16);
      } else {
        unsigned long long ent[OS_NMAX];
#pragma unroll
        for (int j = 0; j < OS_NMAX; ++j)
          if (j < n) ent[j] = slot[row * n + j];
        int first = -1;
#pragma unroll
        for (int j = 0; j < OS_NMAX; ++j)
          if (j < n && (unsigned)(ent[j] >> 32) == epoch) {
            if (first < 0) first = j;
            s_cid[wid][lane][my_cnt++] = (int)(uint32_t)ent[j];
          }
        owned = first == sidx;
        my_row = row;
      }
    }
    own_mask = __ballot_sync(0xffffffffu, owned);
    __syncwarp();
  };
  // producer cursor: lane k of the batch, element pj of cnt + KPRE
  int pk = -1, pj = 0, pcnt = 0;
  int64_t prow = 0;
  auto next_entry = [&]() -> bool {  // advance to the next owned entry
    while (true) {
      if (fb >= fe) return false;
      const unsigned rest = pk < 31 ? own_mask & ~((2u << pk) - 1u) : 0u;
      if (pk >= 0 && rest == 0u) {
        fb += 32;
        pk = -1;
        if (fb >= fe) return false;
        load_batch();
        continue;
      }
      if (pk < 0 && own_mask == 0u) {
        fb += 32;
        if (fb >= fe) return false;
        load_batch();
        continue;
      }
      pk = __ffs(pk < 0 ? own_mask : rest) - 1;
      pcnt = __shfl_sync(0xffffffffu, my_cnt, pk);
      prow = __shfl_sync(0xffffffffu, my_row, pk);
      pj = 0;
      return true;
    }
  };
  bool have = false;
  if (fb < fe) {
    load_batch();
    have = next_entry();
  }
  auto issue = [&](int e) {
    const int sl = e % S;
    const float4* src;
    const bool end = pj + 1 == pcnt + KPRE;
    if (pj < pcnt) {
      src = inbox + (int64_t)s_cid[wid][pk][pj] * D4;
    } else {
      src = pre_base[pj - pcnt] + prow * D4;
    }
    float4* dstp = ring + sl * D4;
#pragma unroll
    for (int v = 0; v < VPT; ++v) cp_async16(dstp + lane + v * 32, src + lane + v * 32);
    if (end) {
      if (lane < pcnt) s_meta[wid][sl].cidx[lane] = s_cid[wid][pk][lane];
      if (lane == 0) {
        s_meta[wid][sl].row = prow;
        s_meta[wid][sl].cnt = pcnt;
      }
    }
    if (lane == 0) s_meta[wid][sl].flags = (pj == 0 ? RS_FIRST : 0) | (pj >= pcnt ? RS_PRE : 0) |
                                           (end ? RS_END : 0);
    __syncwarp();
    if (end) {
      have = next_entry();
    } else {
      ++pj;
    }
  };
  int issued = 0;
#pragma unroll 1
  for (int k = 0; k < F; ++k) {
    if (have) issue(issued++);
    cp_async_commit();
  }
  float4 acc[VPT];
#pragma unroll
  for (int v = 0; v < VPT; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int m = 0; m < issued; ++m) {
    cp_async_wait<F - 1>();
    __syncwarp();
    const int sl = m % S;
    const int flags = s_meta[wid][sl].flags;
    const float4* rowp = ring + sl * D4;
    if (!(flags & RS_PRE)) {
      const bool first = flags & RS_FIRST;
#pragma unroll
      for (int v = 0; v < VPT; ++v)
        acc[v] = f4_add(first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[v], rowp[lane + v * 32]);
    }
    if (flags & RS_END) {
      const int64_t row = s_meta[wid][sl].row;
      const int cnt = s_meta[wid][sl].cnt;
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const int c = lane + v * 32;
        float4 wv = ring[((m - KPRE + 1 + S) % S) * D4 + c];
        float4 av = make_float4(0.f, 0.f, 0.f, 0.f), bv = av;
        if (KPRE > 1) av = ring[((m - KPRE + 2 + S) % S) * D4 + c];
        if (KPRE > 2) bv = ring[((m - KPRE + 3 + S) % S) * D4 + c];
        const float4 g = acc[v];
        opt_update<OPT>(wv.x, av.x, bv.x, g.x, o);
        opt_update<OPT>(wv.y, av.y, bv.y, g.y, o);
        opt_update<OPT>(wv.z, av.z, bv.z, g.z, o);
        opt_update<OPT>(wv.w, av.w, bv.w, g.w, o);
        const int64_t off = row * D4 + c;
        w[off] = wv;
        if (OPT != HP_OPT_SGD) s0[off] = av;
        if (OPT == HP_OPT_ADAM) s1[off] = bv;
        acc[v] = wv;  // the updated row, for the returns below
      }
      for (int j = 0; j < cnt; ++j) {  // pull, fused: back to every contributor
        const int idx = s_meta[wid][sl].cidx[j];
        const int src = idx / (int)L.cap;
        const int64_t ret_row = s_poff[src] + (idx - (int64_t)src * L.cap);
        float4* ret = reinterpret_cast<float4*>(static_cast<char*>(peers.base[src]) + L.ret_off) +
                      ret_row * D4;
#pragma unroll
        for (int v = 0; v < VPT; ++v) ret[lane + v * 32] = acc[v];
      }
    }
    __syncwarp();
    if (have) issue(issued++);
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_last = atomicAdd(&sig.done[1], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      st_release_sys(&SigView(peers.base[r]).applied_flag[L.me], (int)epoch);
    if (threadIdx.x == 0) sig.done[1] = 0;
  }
  HP_SPAN_END(SP_APPLY);
}

// ---- owner, two passes (default). k_owner_scan: one thread per received
// entry (all sources, source-major) resolves id -> slab row and reads the
// row's n slot-table tags; the entry of the lowest-ranked source with a valid
// tag owns the row and writes a merge item {row, cnt} + its contributor list
// (inbox indices in source order) with a warp-aggregated atomic. The whole
// index chain is thus paid once, in parallel, instead of once per entry
// inside the apply loop.
__global__ void __launch_bounds__(256)
k_owner_scan(void* my_win, WinLayout L, const int64_t* __restrict__ part_base, Router route,
             int64_t rows_cap, long long wait_cycles) {
  __shared__ int s_pre[OS_NMAX + 1];
  HP_ENTRY(SP_SCATTER);
  SigView sig(my_win);
  if (wait_cycles > 0) {  // the push wait, folded in (no k_wait launch on the chain)
    const int e = *reinterpret_cast<volatile int*>(sig.epoch);
    for (int s = threadIdx.x; s < L.n; s += blockDim.x) {
      const long long t0 = clock64();
      while (ld_acquire_sys(&sig.push_flag[s]) < e) {
        if (clock64() - t0 > wait_cycles) {
          atomicOr(sig.err, 4);
          break;
        }
        __nanosleep(64);
      }
    }
    __syncthreads();
  }
  char* win = static_cast<char*>(my_win);
  const int64_t* inbox_ids = reinterpret_cast<const int64_t*>(win + L.ids_off);
  const unsigned long long* slot = reinterpret_cast<const unsigned long long*>(win + L.slot_off);
  int2* items = reinterpret_cast<int2*>(win + L.items_off);
  int* cidx = reinterpret_cast<int*>(win + L.cidx_off);
  const int n = L.n;
  // a push wait that timed out (error bit 4) leaves partially written inboxes:
  // merge nothing (0 items) rather than apply them; the runner raises
  if (*reinterpret_cast<volatile int*>(sig.err) & 4) return;
  if (threadIdx.x == 0) {
    int a = 0;
    for (int q = 0; q < n; ++q) {
      s_pre[q] = a;
      a += sig.push_count[q];
    }
    s_pre[n] = a;
  }
  __syncthreads();
  const int E = s_pre[n];
  const unsigned epoch = (unsigned)*sig.epoch;
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t f0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); f0 < E; f0 += wstride) {
    const int f = (int)f0 + lane;
    bool owned = false;
    int row = 0, cnt = 0, sidx = 0;
    unsigned have = 0;
    unsigned long long ent[OS_NMAX];
    if (f < E) {
      while (sidx + 1 < n && f >= s_pre[sidx + 1]) ++sidx;
      const int64_t id = inbox_ids[(int64_t)sidx * L.cap + (f - s_pre[sidx])];
      const int p = route.part(id);
      const int64_t b = part_base[p];
      const int64_t r = b + (id - route.lo(p));
      if (b < 0 || r >= rows_cap) {
        atomicOr(sig.err, 16);
      } else {
        row = (int)r;
#pragma unroll
        for (int j = 0; j < OS_NMAX; ++j)
          if (j < n) ent[j] = slot[r * n + j];
#pragma unroll
        for (int j = 0; j < OS_NMAX; ++j)
          if (j < n && (unsigned)(ent[j] >> 32) == epoch) have |= 1u << j;
        cnt = __popc(have);
        owned = have != 0 && __ffs(have) - 1 == sidx;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, owned);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(sig.own_items, __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (owned) {
      const int pos = base + __popc(m & lanemask_lt());
      items[pos] = make_int2(row, cnt);
      int k = 0;
#pragma unroll
      for (int j = 0; j < OS_NMAX; ++j)
        if (j < n && ((have >> j) & 1u)) cidx[(int64_t)pos * n + k++] = (int)(uint32_t)ent[j];
    }
  }
  HP_SPAN_END(SP_SCATTER);
}

// k_owner_rows: one group of TPI threads (VPT float4 columns each) per merge
// item: the item and its contributor list are one round trip, then the row's
// state and all contributions are loaded together; sums in source order,
// scales, applies, stores the state and returns the updated row into each
// contributor's return buffer (NVLink). No block fences: k_applied (one block,
// next in the stream) fences once at system scope and raises "applied".
template <int OPT, int TPI, int VPT>
__global__ void __launch_bounds__(256, 3)
k_owner_rows(PeerTable peers, void* my_win, WinLayout L, float4* s0, float4* s1, hp_optim o) {
  __shared__ int s_poff[OS_NMAX];
  HP_ENTRY(SP_APPLY);
  SigView sig(my_win);
  char* win = static_cast<char*>(my_win);
  float4* w = reinterpret_cast<float4*>(win + L.w_off);
  const float4* inbox = reinterpret_cast<const float4*>(win + L.rows_off);
  const int2* items = reinterpret_cast<const int2*>(win + L.items_off);
  const int* cidx_all = reinterpret_cast<const int*>(win + L.cidx_off);
  const int n = L.n, D4 = L.D4;
  if (threadIdx.x < n) s_poff[threadIdx.x] = sig.push_off[threadIdx.x];
  __syncthreads();
  const int NI = *sig.own_items;
  const int lane = threadIdx.x & 31, q = threadIdx.x % TPI;
  constexpr int GPB = 256 / TPI;
  // one item per group, many waves (blocks past the item count exit at once and
  // take no part in the last-block election); with a capped grid the group
  // loops, the next descriptor loaded while this item streams
  if ((int)blockIdx.x * GPB >= NI) return;
  const int istride = gridDim.x * GPB;
  int it = blockIdx.x * GPB + threadIdx.x / TPI;
  int2 item_n = make_int2(0, 0);
  int myc_n = 0;
  if (it < NI) {
    item_n = items[it];
    myc_n = lane < n ? cidx_all[(int64_t)it * n + lane] : 0;
  }
  for (; it < NI; it += istride) {
    const int2 item = item_n;
    const int myc = myc_n;
    const int64_t row = item.x;
    const int cnt = item.y;
    float4 wv[VPT], av[VPT], bv[VPT], g[VPT];
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c = q + v * TPI;
      const int64_t off = row * D4 + c;
      wv[v] = av[v] = bv[v] = g[v] = z;
      if (c < D4) {
        wv[v] = w[off];
        if (OPT != HP_OPT_SGD) av[v] = s0[off];
        if (OPT == HP_OPT_ADAM) bv[v] = s1[off];
      }
    }
    for (int j0 = 0; j0 < cnt; j0 += 2) {  // contributions, in source order
      float4 x[2][VPT];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int idx = __shfl_sync(0xffffffffu, myc, (j0 + u) & 31);
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (j0 + u < cnt && q + v * TPI < D4) x[u][v] = inbox[(int64_t)idx * D4 + q + v * TPI];
      }
      if (j0 == 0 && it + istride < NI) {  // prefetch the next descriptor
        item_n = items[it + istride];
        myc_n = lane < n ? cidx_all[(int64_t)(it + istride) * n + lane] : 0;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (j0 + u < cnt) g[v] = f4_add(g[v], x[u][v]);
    }
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c = q + v * TPI;
      if (c >= D4) continue;
      opt_update<OPT>(wv[v].x, av[v].x, bv[v].x, g[v].x, o);
      opt_update<OPT>(wv[v].y, av[v].y, bv[v].y, g[v].y, o);
      opt_update<OPT>(wv[v].z, av[v].z, bv[v].z, g[v].z, o);
      opt_update<OPT>(wv[v].w, av[v].w, bv[v].w, g[v].w, o);
      const int64_t off = row * D4 + c;
      w[off] = wv[v];
      if (OPT != HP_OPT_SGD) s0[off] = av[v];
      if (OPT == HP_OPT_ADAM) s1[off] = bv[v];
    }
    for (int j = 0; j < cnt; ++j) {  // pull, fused: back to every contributor's send slot
      const int idx = __shfl_sync(0xffffffffu, myc, j);
      const int src = idx / (int)L.cap;
      const int64_t ret_row = s_poff[src] + (idx - (int64_t)src * L.cap);
      float4* ret = reinterpret_cast<float4*>(static_cast<char*>(peers.base[src]) + L.ret_off) +
                    ret_row * D4;
#pragma unroll
      for (int v = 0; v < VPT; ++v)
        if (q + v * TPI < D4) ret[q + v * TPI] = wv[v];
    }
  }
  HP_SPAN_END(SP_APPLY);
}

// After k_owner_rows (stream order): one system fence covering every store of
// the apply, then "applied" at every rank; resets the item counter.
__global__ void k_applied(PeerTable peers, void* my_win, WinLayout L) {
  HP_ENTRY(SP_APPLIED);
  SigView sig(my_win);
  __threadfence_system();
  const int epoch = *sig.epoch;
  for (int r = threadIdx.x; r < L.n; r += blockDim.x)
    st_release_sys(&SigView(peers.base[r]).applied_flag[L.me], epoch);
  if (threadIdx.x == 0) *sig.own_items = 0;
  HP_SPAN_END(SP_APPLIED);
}

}  // namespace

// ---- forward pull (a worker's lookup of rows homed anywhere): one warp per id
// reads the row straight out of its owner's slab over NVLink (every slab lives
// in its rank's peer-mapped window) — no owner participation. Dropped ids give
// zero rows. Callers order it after the previous step's "applied" (the stitch
// waited for every owner) and before their own next push, so no owner can be
// updating the rows being read (an owner applies step i+1 only after every
// source, this one included, pushed step i+1).
__global__ void __launch_bounds__(256)
k_peer_pull(PeerTable peers, WinLayout L, const int64_t* __restrict__ ids, int64_t T, Router route,
            int64_t V, const int32_t* __restrict__ owner, const int64_t* __restrict__ glob_base,
            float4* __restrict__ out) {
  HP_ENTRY(SP_COPY);
  const int lane = threadIdx.x & 31;
  const int D4 = L.D4;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < T;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t id = ids[r];
    const float4* src = nullptr;
    if (id >= 0 && id < V) {
      const int p = route.part(id);
      const int64_t row = glob_base[p] + (id - route.lo(p));
      src = reinterpret_cast<const float4*>(static_cast<const char*>(peers.base[owner[p]]) + L.w_off) +
            row * D4;
    }
    for (int c0 = lane; c0 < D4; c0 += 32 * 4) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u;
        x[u] = (src && c < D4) ? src[c] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + 32 * u;
        if (c < D4) out[r * D4 + c] = x[u];
      }
    }
  }
  HP_SPAN_END(SP_COPY);
}

// Spin-wait budget (cycles) before a wait gives up and raises an error bit:
// hp_debug_set_wait_timeout (> 0), else HP_WAIT_TIMEOUT_CYCLES, else ~2 s.
long long g_wait_cycles = 0;
long long wait_budget() {
  if (g_wait_cycles > 0) return g_wait_cycles;
  static long long v = [] {
    const char* e = getenv("HP_WAIT_TIMEOUT_CYCLES");
    return e ? atoll(e) : 4000000000LL;  // ~2 s at 1.9 GHz
  }();
  return v;
}

HP_SPAN_SETTER(set_spans_p2p)

}  // namespace hp

using namespace hp;

// Opaque exchange state for one table (declared in include/hybridpath.h).
struct hp_xchg_s {
  WinLayout L;
  int64_t rows_cap, bytes;
  void* win;          // own window
  PeerTable peers;    // mapped windows (own = win)
  uint64_t ipc_mask;  // peers mapped with cudaIpcOpenMemHandle (closed on destroy)
};

extern "C" {

size_t hp_xchg_window_bytes(int32_t n, int32_t D, int64_t cap, int64_t rows_cap) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  return al(SIG_INTS * 4) + al((size_t)rows_cap * D * 4) + al((size_t)n * cap * 8) +
         al((size_t)n * cap * D * 4) + al((size_t)cap * D * 4) + al((size_t)rows_cap * n * 8) +
         al((size_t)n * cap * 8) + al((size_t)n * cap * n * 4);
}

int hp_xchg_create(hp_xchg_t* out, int32_t n, int32_t me, int32_t D, int64_t cap, int64_t rows_cap,
                   void* ipc_handle_out /* 64 bytes */, void** w_out) {
  // n <= HP_CHUNK: the owner's source-order sum is then one sequential group of
  // the summation tree (oracle.grouped_tree_sum)
  HP_REQUIRE(out && ipc_handle_out && w_out && n >= 1 && n <= HP_CHUNK && me >= 0 && me < n,
             "bad xchg args (1 <= n <= 16)");
  HP_REQUIRE(D % 4 == 0 && D >= 4 && D <= 2048 && cap >= 1 && rows_cap >= 1, "bad xchg shape");
  auto* x = new hp_xchg_s{};
  auto al = [](int64_t v) { return (v + 255) & ~(int64_t)255; };
  WinLayout& L = x->L;
  L.n = n;
  L.me = me;
  L.D4 = D / 4;
  L.cap = cap;
  x->rows_cap = rows_cap;
  L.w_off = al(SIG_INTS * 4);
  L.ids_off = L.w_off + al(rows_cap * D * 4);
  L.rows_off = L.ids_off + al((int64_t)n * cap * 8);
  L.ret_off = L.rows_off + al((int64_t)n * cap * D * 4);
  L.slot_off = L.ret_off + al(cap * D * 4);
  L.items_off = L.slot_off + al(rows_cap * n * 8);
  L.cidx_off = L.items_off + al((int64_t)n * cap * 8);
  x->bytes = L.cidx_off + al((int64_t)n * cap * n * 4);
  cudaError_t e = cudaMalloc(&x->win, x->bytes);
  if (e != cudaSuccess) {
    delete x;
    return cuda_fail(e, "cudaMalloc(window)");
  }
  HP_CUDA(cudaMemset(x->win, 0, SIG_INTS * 4));
  HP_CUDA(cudaMemset(static_cast<char*>(x->win) + L.slot_off, 0, (size_t)rows_cap * n * 8));
  cudaIpcMemHandle_t h;
  HP_CUDA(cudaIpcGetMemHandle(&h, x->win));
  static_assert(sizeof(h) == 64, "IPC handle size");
  memcpy(ipc_handle_out, &h, sizeof(h));
  for (int r = 0; r < 64; ++r) x->peers.base[r] = nullptr;
  x->peers.base[me] = x->win;
  *w_out = static_cast<char*>(x->win) + L.w_off;
  *out = x;
  return HP_OK;
}

int hp_xchg_open_peer(hp_xchg_t x, int32_t rank, const void* ipc_handle) {
  HP_REQUIRE(x && rank >= 0 && rank < x->L.n && ipc_handle, "bad peer args");
  if (rank == x->L.me) return HP_OK;
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  void* p = nullptr;
  HP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  x->peers.base[rank] = p;
  x->ipc_mask |= 1ull << rank;
  return HP_OK;
}

// Single-process emulation of n ranks (tests on one GPU): the windows are
// plain device allocations of this process, so a peer is set from its raw
// window address instead of a cudaIpc handle. Same kernels, same protocol.
int hp_xchg_window_ptr(hp_xchg_t x, void** out) {
  HP_REQUIRE(x && out, "NULL argument");
  *out = x->win;
  return HP_OK;
}

int hp_xchg_set_peer_ptr(hp_xchg_t x, int32_t rank, void* window) {
  HP_REQUIRE(x && rank >= 0 && rank < x->L.n && window, "bad peer args");
  if (rank == x->L.me) return HP_OK;
  HP_REQUIRE(!((x->ipc_mask >> rank) & 1ull), "peer already mapped by IPC");
  x->peers.base[rank] = window;
  return HP_OK;
}

int hp_xchg_destroy(hp_xchg_t x) {
  if (!x) return HP_OK;
  for (int r = 0; r < x->L.n; ++r)
    if (r != x->L.me && ((x->ipc_mask >> r) & 1ull)) cudaIpcCloseMemHandle(x->peers.base[r]);
  cudaFree(x->win);
  delete x;
  return HP_OK;
}

// Worker K1+K2 (index half of hp_xchg_push): dedup + route ids[T] into a send
// plan left in ws; outputs send_ids[U], inv[T], dest_counts[n], n_uniq.
int hp_xchg_plan(hp_xchg_t x, const int64_t* ids, int64_t T, int64_t V, int32_t P,
                 const int32_t* owner, const int64_t* glob_base, int64_t* send_ids, int32_t* inv,
                 int32_t* dest_counts, int32_t* n_uniq, void* ws, size_t ws_bytes, void* stream) {
  HP_REQUIRE(x && owner && glob_base && send_ids && inv && dest_counts && n_uniq, "NULL argument");
  HP_REQUIRE(T <= x->L.cap, "more ids than the inbox capacity");
  HP_REQUIRE(T == 0 || ids, "NULL ids");
  DedupPlan pl;
  int rc = carve_plan(&pl, ws, ws_bytes, T, x->L.D4 * 4, V, P, x->L.n);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = build_plan(pl, ids, owner, nullptr, send_ids, nullptr, inv, dest_counts, n_uniq, st);
  if (rc || T == 0) return rc;
  k_send_info<<<grid_for(T, 256, sm_count() * 4), 256, 0, st>>>(
      send_ids, dest_counts, n_uniq, glob_base, Router(V, P), x->L, pl.send_info, T);
  HP_LAUNCHED(1, "k_send_info");
  return HP_OK;
}

// Worker K1 values + K3, fused: with the plan in ws (hp_xchg_plan, same T / V / P),
// reduce vals[T, D] and store every summed row straight into its owner's inbox
// over NVLink; the last block publishes counts / offsets / epoch at every owner.
int hp_xchg_push_plan(hp_xchg_t x, const float* vals, int64_t T, int64_t V, int32_t P,
                      const int64_t* send_ids, const int32_t* dest_counts,
                      const int64_t* glob_base, void* ws, size_t ws_bytes, void* stream,
                      void* side_stream) {
  HP_REQUIRE(x && send_ids && dest_counts && glob_base, "NULL argument");
  HP_REQUIRE(T == 0 || vals, "NULL vals");
  DedupPlan pl;
  int rc = carve_plan(&pl, ws, ws_bytes, T, x->L.D4 * 4, V, P, x->L.n);
  if (rc) return rc;
  restore_sorted_pos(pl);
  EpiPush epi{x->peers, x->L, dest_counts, send_ids, pl.send_info, x->win};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (side_stream != nullptr && T > 0 && pl.reorder && !pl.fused && pl.nw <= 0) {
    // long-first items: the short items' reduce + peer stores fork onto
    // side_stream; the long chunks -> k_combine stay on stream; after the
    // join one k_publish (its system fence covers both branches' stores)
    cudaStream_t ss = static_cast<cudaStream_t>(side_stream);
    cudaEvent_t fork = push_event(0), join = push_event(1);
    HP_CUDA(cudaEventRecord(fork, st));
    HP_CUDA(cudaStreamWaitEvent(ss, fork, 0));
    DedupPlan ps = pl, pg = pl;
    ps.part = 2;
    pg.part = 1;
    if ((rc = launch_reduce(ps, vals, epi, ss))) return rc;
    HP_CUDA(cudaEventRecord(join, ss));
    if ((rc = launch_reduce(pg, vals, epi, st))) return rc;  // no publication for part 1
    HP_CUDA(cudaStreamWaitEvent(st, join, 0));
    launch_k(k_publish<EpiPush>, dim3(1), dim3(64), 0, st, epi);
    HP_LAUNCHED(1, "k_publish");
    return HP_OK;
  }
  pl.T = std::max<int64_t>(T, 1);  // launch even for T == 0: k_publish carries the publication
  return launch_reduce(pl, vals, epi, st);
}

// Worker, fused K1+K2+K3 = hp_xchg_plan + hp_xchg_push_plan.
int hp_xchg_push(hp_xchg_t x, const int64_t* ids, const float* vals, int64_t T, int64_t V,
                 int32_t P, const int32_t* owner, const int64_t* glob_base, int64_t* send_ids,
                 int32_t* inv, int32_t* dest_counts, int32_t* n_uniq, void* ws, size_t ws_bytes,
                 void* stream) {
  int rc = hp_xchg_plan(x, ids, T, V, P, owner, glob_base, send_ids, inv, dest_counts, n_uniq, ws,
                        ws_bytes, stream);
  if (rc) return rc;
  return hp_xchg_push_plan(x, vals, T, V, P, send_ids, dest_counts, glob_base, ws, ws_bytes,
                           stream, nullptr);
}

// Owner: wait for every source's push, merge in source order, apply to the
// slab, return the updated rows to the contributors, signal "applied".
int hp_xchg_wait(hp_xchg_t x, int32_t which, void* stream) {
  HP_REQUIRE(x && (which == 0 || which == 1), "bad wait arguments");
  launch_k(k_wait, dim3(1), dim3(64), 0, static_cast<cudaStream_t>(stream), x->win, which, x->L.n, wait_budget(),
           which ? SP_WAIT_APPLIED : SP_WAIT_PUSH, 0);
  HP_LAUNCHED(1, "k_wait");
  return HP_OK;
}

extern "C++" {
template <int OPT, int TPI, int VPT>
void launch_owner_apply(const hp_xchg_s* x, const hp_slab& slab, const hp_optim& opt,
                        cudaStream_t st) {
  const int64_t total = (int64_t)x->L.n * x->L.cap;
  const int blocks = grid_for(total, 256 / TPI, sm_count() * (VPT >= 4 ? 2 : 3));  // one wave
  launch_k(k_owner_apply<OPT, TPI, VPT>, dim3(blocks), dim3(256), 0, st, 
      x->peers, x->win, x->L, slab.part_base, Router(slab.V, slab.P),
      reinterpret_cast<float4*>(slab.s0), reinterpret_cast<float4*>(slab.s1), opt, x->rows_cap);
}

template <int OPT, int VPT>
void launch_owner_stream(const hp_xchg_s* x, const hp_slab& slab, const hp_optim& opt,
                         cudaStream_t st) {
  constexpr int S = VPT == 1 ? 16 : (VPT == 2 ? 12 : (VPT == 4 ? 8 : 6));
  constexpr size_t smem = (size_t)4 * S * VPT * 32 * sizeof(float4);
  auto kern = k_owner_stream<OPT, VPT, S>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  const int ctas = std::max(1, std::min(g_rs_ctas, (int)((160u << 10) / smem)));
  launch_k(kern, dim3(sm_count() * ctas), dim3(128), smem, st, x->peers, x->win, x->L,
           slab.part_base, Router(slab.V, slab.P), reinterpret_cast<float4*>(slab.s0),
           reinterpret_cast<float4*>(slab.s1), opt, x->rows_cap);
}

template <int OPT, int TPI, int VPT>
void launch_owner_rows(const hp_xchg_s* x, const hp_slab& slab, const hp_optim& opt,
                       cudaStream_t st, bool wait) {
  const int64_t total = (int64_t)x->L.n * x->L.cap;
  launch_k(k_owner_scan, dim3(grid_for(total, 256, sm_count() * 8)), dim3(256), 0, st, x->win, x->L,
           slab.part_base, Router(slab.V, slab.P), x->rows_cap, wait ? wait_budget() : 0LL);
  const int blocks = grid_for(total, 256 / TPI, g_owner_waves ? 1 << 30 : sm_count() * 3);
  launch_k(k_owner_rows<OPT, TPI, VPT>, dim3(blocks), dim3(256), 0, st, x->peers, x->win, x->L,
           reinterpret_cast<float4*>(slab.s0), reinterpret_cast<float4*>(slab.s1), opt);
  launch_k(k_applied, dim3(1), dim3(64), 0, st, x->peers, x->win, x->L);
}

template <int OPT>
void dispatch_owner_apply(const hp_xchg_s* x, const hp_slab& slab, const hp_optim& opt, int D4,
                          cudaStream_t st, bool wait) {
  if (g_owner_stream == 2) {
    if (D4 <= 32) launch_owner_rows<OPT, 32, 1>(x, slab, opt, st, wait);
    else if (D4 <= 64) launch_owner_rows<OPT, 32, 2>(x, slab, opt, st, wait);
    else if (D4 <= 128) launch_owner_rows<OPT, 64, 2>(x, slab, opt, st, wait);
    else if (D4 <= 256) launch_owner_rows<OPT, 128, 2>(x, slab, opt, st, wait);  // spill-free at D = 1024
    else launch_owner_rows<OPT, 256, 2>(x, slab, opt, st, wait);
    return;
  }
  if (wait) hp_xchg_wait(const_cast<hp_xchg_s*>(x), 0, st);
  if (g_owner_stream == 1) {
    switch (D4) {
      case 32: return launch_owner_stream<OPT, 1>(x, slab, opt, st);
      case 64: return launch_owner_stream<OPT, 2>(x, slab, opt, st);
      case 128: return launch_owner_stream<OPT, 4>(x, slab, opt, st);
      case 256: return launch_owner_stream<OPT, 8>(x, slab, opt, st);
      default: break;
    }
  }
  if (D4 <= 32) launch_owner_apply<OPT, 32, 1>(x, slab, opt, st);
  else if (D4 <= 64) launch_owner_apply<OPT, 32, 2>(x, slab, opt, st);
  else if (D4 <= 128) launch_owner_apply<OPT, 64, 2>(x, slab, opt, st);
  else if (D4 <= 256) launch_owner_apply<OPT, 64, 4>(x, slab, opt, st);
  else launch_owner_apply<OPT, 128, 4>(x, slab, opt, st);
}
}  // extern "C++"

int hp_xchg_merge_apply(hp_xchg_t x, hp_slab slab, hp_optim opt, int32_t wait, void* stream) {
  HP_REQUIRE(x && slab.part_base, "NULL argument");
  HP_REQUIRE(slab.D == x->L.D4 * 4, "slab width differs from the exchange");
  HP_REQUIRE(opt.kind == HP_OPT_SGD || slab.s0, "optimizer state s0 is NULL");
  HP_REQUIRE(opt.kind != HP_OPT_ADAM || slab.s1, "Adam state s1 is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the push wait: folded into k_owner_scan (default owner kernels), else k_wait
  const int D4 = x->L.D4;
  switch (opt.kind) {
    case HP_OPT_SGD: dispatch_owner_apply<HP_OPT_SGD>(x, slab, opt, D4, st, wait != 0); break;
    case HP_OPT_ADAGRAD: dispatch_owner_apply<HP_OPT_ADAGRAD>(x, slab, opt, D4, st, wait != 0); break;
    default: dispatch_owner_apply<HP_OPT_ADAM>(x, slab, opt, D4, st, wait != 0);
  }
  HP_LAUNCHED(g_owner_stream == 2 ? 3 : 1, "owner merge/apply");
  return HP_OK;
}

// Worker: wait for every owner's apply, then out[t] = returned row of send slot inv[t].
int hp_xchg_stitch(hp_xchg_t x, const int32_t* inv, int64_t T, float* out, int32_t wait,
                   void* stream) {
  HP_REQUIRE(x && (T == 0 || (inv && out)), "NULL argument");
  if (wait) {  // also with no ids: the next push must follow every owner's apply
    int rc = hp_xchg_wait(x, 1, stream);
    if (rc) return rc;
  }
  if (T == 0) return HP_OK;
  const float* ret = reinterpret_cast<const float*>(static_cast<char*>(x->win) + x->L.ret_off);
  return hp_stitch(ret, inv, T, x->L.D4 * 4, out, stream);
}

// Debug: copy the window's signal words (SIG_INTS ints) to host memory (syncs).
int hp_xchg_debug_sig(hp_xchg_t x, int32_t* host_out, void* stream) {
  HP_REQUIRE(x && host_out, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_CUDA(cudaMemcpyAsync(host_out, x->win, SIG_INTS * 4, cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  return HP_OK;
}

// Rows received from each source in the last push (device copy, stream-ordered).
int hp_xchg_recv_counts(hp_xchg_t x, int32_t* out_dev, void* stream) {
  HP_REQUIRE(x && out_dev, "NULL argument");
  SigView sig(x->win);
  HP_CUDA(cudaMemcpyAsync(out_dev, sig.push_count, 4 * (size_t)x->L.n, cudaMemcpyDeviceToDevice,
                          static_cast<cudaStream_t>(stream)));
  return HP_OK;
}

int hp_xchg_pull(hp_xchg_t x, const int64_t* ids, int64_t T, int64_t V, int32_t P,
                 const int32_t* owner, const int64_t* glob_base, float* out, void* stream) {
  HP_REQUIRE(x && owner && glob_base && (T == 0 || (ids && out)), "NULL argument");
  HP_REQUIRE(V >= 1 && V < (int64_t(1) << 31) && P >= 1 && P <= V, "bad V / P");
  if (T == 0) return HP_OK;
  for (int r = 0; r < x->L.n; ++r) HP_REQUIRE(x->peers.base[r], "a peer window is not mapped");
  launch_k(k_peer_pull, dim3(grid_for(T, 8, sm_count() * 8)), dim3(256), 0,
           static_cast<cudaStream_t>(stream), x->peers, x->L, ids, T, Router(V, P), V, owner,
           glob_base, reinterpret_cast<float4*>(out));
  HP_LAUNCHED(1, "k_peer_pull");
  return HP_OK;
}

int hp_xchg_stitch_plan(hp_xchg_t x, const void* ws, size_t ws_bytes, int64_t T, int64_t V,
                        int32_t P, float* out, int32_t wait, void* stream) {
  HP_REQUIRE(x && ws, "NULL argument");
  SigView sig(x->win);
  const float* ret = reinterpret_cast<const float*>(static_cast<char*>(x->win) + x->L.ret_off);
  StitchWait w{wait ? sig.applied_flag : nullptr, sig.epoch, sig.err, x->L.n, wait_budget()};
  if (T == 0) {  // no rows, but the next push must still follow every owner's apply
    return wait ? hp_xchg_wait(x, 1, stream) : HP_OK;
  }
  return plan_stitch(ws, ws_bytes, T, x->L.D4 * 4, V, P, ret, out,
                     static_cast<cudaStream_t>(stream), 0, wait ? &w : nullptr);
}

int hp_xchg_ret_ptr(hp_xchg_t x, float** out) {
  HP_REQUIRE(x && out, "NULL argument");
  *out = reinterpret_cast<float*>(static_cast<char*>(x->win) + x->L.ret_off);
  return HP_OK;
}

// Device address of the exchange's error word (for hp_err_collect).
int hp_xchg_err_ptr(hp_xchg_t x, const int32_t** out) {
  HP_REQUIRE(x && out, "NULL argument");
  *out = SigView(x->win).err;
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

// ============================================================================
// K7 over peer memory: dense gradient allreduce fused with scale + cast.
//
// Rank r owns chunk r of the S elements. Phase 1 (k_ar_scatter): every rank
// stores chunk c != me of its own gradient into rank c's reduce slot [me][*]
// (NVLink stores; the gradient is read locally, in place, no staging copy).
// Phase 2 (k_ar_reduce_gather): rank c sums the n contributions of its chunk
// in source-rank order (its own read from grad; deterministic,
// bit-reproducible), multiplies by scale, casts, and stores the result into
// every rank's output. Each phase is published by a one-block k_signal (one
// system fence, cumulative over the stream's earlier kernels) and ordered
// across GPUs by one-block k_wait kernels. Both phases run in nb buckets
// (pieces of every chunk), so the waits of one bucket overlap the others.
// Per rank NVLink bytes: (n-1)/n * S * (4 + out_bytes).
// ============================================================================
namespace hp {
namespace {

constexpr int AR_MAXN = 32;
struct ArLayout {
  int64_t S, S_real, chunk, slots_off, out_off;  // S = S_real padded to a multiple of 4n
  int n, me, out_bytes;
  int in_bytes;  // 4 = fp32 gradients, 2 = bf16 (SM mode; slots then hold bf16, half the NVLink bytes)
  // chunk of rank r = float4 range [off4[r], off4[r+1]) (uniform S/n unless
  // hp_dar_set_split weighted it); source s's slot at every rank starts at s * sstride4
  int64_t sstride4;
  int64_t off4[AR_MAXN + 1];
};

// Bucket bk of nb: every chunk is cut into nb pieces, [c4*bk/nb, c4*(bk+1)/nb)
// float4 of it; bucket bk's scatter, reduce and gather only touch piece bk.
__host__ __device__ __forceinline__ int64_t ar_piece(int64_t c4, int bk, int nb) {
  return c4 * bk / nb;
}

// Four gradient elements as one vector: float4 (fp32) or uint2 (4 x bf16).
template <typename InT> struct Vec4;
template <> struct Vec4<float> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  static __device__ __forceinline__ float4 f32(T v) { return v; }
  static __device__ __forceinline__ T ld(const T* p) { return ldg_stream(p); }
};
template <> struct Vec4<__nv_bfloat16> {
  using T = uint2;
  static __device__ __forceinline__ T zero() { return make_uint2(0u, 0u); }
  static __device__ __forceinline__ float4 f32(T v) {  // exact widening
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  static __device__ __forceinline__ T ld(const T* p) {
    T v;
    asm volatile("ld.global.cs.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
  }
};

// blockIdx.y = destination peer (my own chunk is not copied: the reduce reads
// my contribution straight from grad); 4 vectors in flight per thread. bf16
// gradients travel as bf16 (slot s of a rank holds them at the same byte
// offset as fp32 would, half of it used).
template <typename InT, int U = 4>
__global__ void __launch_bounds__(256)
k_ar_scatter(PeerTable peers, ArLayout A, const void* __restrict__ grad_v, int bk, int nb) {
  using V = Vec4<InT>;
  using VT = typename V::T;
  HP_ENTRY(SP_AR_SCATTER);
  const int c = (int)blockIdx.y < A.me ? (int)blockIdx.y : (int)blockIdx.y + 1;
  const int64_t b4 = A.off4[c], c4 = A.off4[c + 1] - b4, real4 = A.S_real >> 2;
  const int64_t p0 = ar_piece(c4, bk, nb), p1 = ar_piece(c4, bk + 1, nb);
  const VT* src = static_cast<const VT*>(grad_v) + b4;
  VT* dst = reinterpret_cast<VT*>(static_cast<char*>(peers.base[c]) + A.slots_off +
                                  (int64_t)A.me * A.sstride4 * 16);
  const int64_t lim = min(p1, max((int64_t)0, real4 - b4));  // real elements here
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = p0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < p1; j0 += U * stride) {
    VT v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      v[u] = j < lim ? V::ld(src + j) : V::zero();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < p1) dst[j] = v[u];
    }
  }
  // no per-block fence: k_signal (next in the stream) fences once at system
  // scope, cumulatively over every peer store of this kernel, then publishes
  HP_SPAN_END(SP_AR_SCATTER);
}

// TMA variant of the scatter (fp32; hp_debug_set_dar_tma): each CTA moves its
// pieces of the peer chunk global -> shared -> peer slot with bulk copies
// (double-buffered, one elected thread), so a few CTAs saturate NVLink and the
// rest of the SMs stay with the sparse tables. The slot padding past S_real is
// never written (zero since the window's creation).
constexpr int AR_TMA_F4 = 2048;  // 32 KB per piece
__global__ void __launch_bounds__(32)
k_ar_scatter_tma(PeerTable peers, ArLayout A, const float4* __restrict__ grad) {
  extern __shared__ __align__(128) float4 s_buf[];  // [2][AR_TMA_F4]
  __shared__ uint64_t s_bar[2];
  HP_ENTRY(SP_AR_SCATTER);
  const int c = (int)blockIdx.y < A.me ? (int)blockIdx.y : (int)blockIdx.y + 1;
  const int64_t b4 = A.off4[c], c4 = A.off4[c + 1] - b4, real4 = A.S_real >> 2;
  const int64_t lim = min(c4, max((int64_t)0, real4 - b4));
  float4* dst = reinterpret_cast<float4*>(static_cast<char*>(peers.base[c]) + A.slots_off) +
                (int64_t)A.me * A.sstride4;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t ph[2] = {0u, 0u};
    int k = 0;
    for (int64_t lo = (int64_t)blockIdx.x * AR_TMA_F4; lo < lim;
         lo += (int64_t)gridDim.x * AR_TMA_F4, ++k) {
      const int b = k & 1;
      const uint32_t bytes = (uint32_t)min((int64_t)AR_TMA_F4, lim - lo) * 16u;
      bulk_wait_read1();  // the store that last read buffer b (two pieces ago) is done reading
      mbar_expect_tx(&s_bar[b], bytes);
      bulk_g2s(s_buf + b * AR_TMA_F4, grad + b4 + lo, bytes, &s_bar[b]);
      mbar_wait(&s_bar[b], ph[b]);
      ph[b] ^= 1u;
      bulk_s2g(dst + lo, s_buf + b * AR_TMA_F4, bytes);
      bulk_commit();
    }
    bulk_wait0();  // every piece written before the kernel ends (k_signal publishes next)
    fence_proxy_async_global();
  }
  HP_SPAN_END(SP_AR_SCATTER);
}

// TMA variant of the reduce/gather (fp32 in and out; hp_debug_set_dar_rg_tma):
// per 16 KB piece of my chunk, the n contributions are bulk-loaded into shared
// memory in source-rank order (double-buffered: contribution s+1 lands while
// s is added), summed per column by 128 threads from +0.0 in rank order,
// scaled, staged in shared memory and bulk-stored into every rank's output.
constexpr int AR_RG_F4 = 1024;  // 16 KB per piece
__global__ void __launch_bounds__(128)
k_ar_rg_tma(PeerTable peers, void* my_win, ArLayout A, const float4* __restrict__ grad, float scale) {
  extern __shared__ __align__(128) float4 s_rg[];  // [2][AR_RG_F4] loads, [AR_RG_F4] result
  __shared__ uint64_t s_bar[2];
  HP_ENTRY(SP_AR_RG);
  const int64_t b4 = A.off4[A.me], c4 = A.off4[A.me + 1] - b4;
  const int64_t own_lim = min(c4, max((int64_t)0, (A.S_real >> 2) - b4));
  const char* slots = static_cast<const char*>(my_win) + A.slots_off;
  float4* res = s_rg + 2 * AR_RG_F4;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  __syncthreads();
  uint32_t ph[2] = {0u, 0u};
  int ld = 0;  // loads issued (buffer = ld & 1)
  constexpr int PER = AR_RG_F4 / 128;
#pragma unroll 1
  for (int64_t lo = (int64_t)blockIdx.x * AR_RG_F4; lo < c4; lo += (int64_t)gridDim.x * AR_RG_F4) {
    const int64_t len = min((int64_t)AR_RG_F4, c4 - lo);
    // source s's piece: own gradient (real part; zeros past S_real) or slot s
    auto issue = [&](int s, int b) {
      if (threadIdx.x != 0) return;
      const float4* src;
      int64_t nbytes;
      if (s == A.me) {
        src = grad + b4 + lo;
        nbytes = max((int64_t)0, min(len, own_lim - lo)) * 16;
      } else {
        src = reinterpret_cast<const float4*>(slots + (int64_t)s * A.sstride4 * 16) + lo;
        nbytes = len * 16;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic reads of b
      mbar_expect_tx(&s_bar[b], (uint32_t)nbytes);
      if (nbytes > 0) bulk_g2s(s_rg + b * AR_RG_F4, src, (uint32_t)nbytes, &s_bar[b]);
    };
    float4 acc[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    issue(0, ld & 1);
#pragma unroll 1
    for (int s = 0; s < A.n; ++s) {
      const int b = (ld + s) & 1;
      if (s + 1 < A.n) issue(s + 1, (ld + s + 1) & 1);
      mbar_wait(&s_bar[b], ph[b]);
      ph[b] ^= 1u;
      const int64_t have = s == A.me ? max((int64_t)0, min(len, own_lim - lo)) : len;
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int j = threadIdx.x + k * 128;
        if (j < len) acc[k] = f4_add(acc[k], j < have ? s_rg[b * AR_RG_F4 + j] : make_float4(0.f, 0.f, 0.f, 0.f));
      }
      __syncthreads();  // buffer b is consumed before it is reloaded (contribution s+2)
    }
    ld += A.n;
    if (threadIdx.x == 0) bulk_wait_read0();  // the previous piece's stores have read `res`
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int j = threadIdx.x + k * 128;
      if (j < len) {
        float4 v = acc[k];
        v.x = __fmul_rn(v.x, scale);
        v.y = __fmul_rn(v.y, scale);
        v.z = __fmul_rn(v.z, scale);
        v.w = __fmul_rn(v.w, scale);
        res[j] = v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int r = 0; r < A.n; ++r)
        bulk_s2g(reinterpret_cast<float4*>(static_cast<char*>(peers.base[r]) + A.out_off) + b4 + lo,
                 res, (uint32_t)(len * 16));
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) {
    bulk_wait0();
    fence_proxy_async_global();
  }
  HP_SPAN_END(SP_AR_RG);
}

template <typename OutT>
__device__ __forceinline__ void put4(void* base, int64_t i4, float4 v);
template <>
__device__ __forceinline__ void put4<float>(void* base, int64_t i4, float4 v) {
  reinterpret_cast<float4*>(base)[i4] = v;
}
template <>
__device__ __forceinline__ void put4<__nv_bfloat16>(void* base, int64_t i4, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  reinterpret_cast<uint2*>(base)[i4] = u;
}

template <typename OutT, typename InT, int U = 2>
__global__ void __launch_bounds__(256)
k_ar_reduce_gather(PeerTable peers, void* my_win, ArLayout A, const void* __restrict__ grad_v,
                   float scale, int bk, int nb) {
  using V = Vec4<InT>;
  using VT = typename V::T;
  HP_ENTRY(SP_AR_RG);
  const int64_t b4 = A.off4[A.me], c4 = A.off4[A.me + 1] - b4;
  const int64_t p0 = ar_piece(c4, bk, nb), p1 = ar_piece(c4, bk + 1, nb);
  const int64_t own_lim = min(p1, max((int64_t)0, (A.S_real >> 2) - b4));
  const char* slots = static_cast<const char*>(my_win) + A.slots_off;
  const VT* mine = static_cast<const VT*>(grad_v) + b4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = p0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < p1; j0 += U * stride) {
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < p1)
        for (int s = 0; s < A.n; ++s) {  // source-rank order; my own from grad (fp32 sums)
          const float4 x =
              s == A.me ? (j < own_lim ? V::f32(V::ld(mine + j)) : make_float4(0.f, 0.f, 0.f, 0.f))
                        : V::f32(V::ld(reinterpret_cast<const VT*>(slots + (int64_t)s * A.sstride4 * 16) + j));
          acc[u] = f4_add(acc[u], x);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      if (j >= p1) continue;
      float4 v = acc[u];
      v.x = __fmul_rn(v.x, scale);
      v.y = __fmul_rn(v.y, scale);
      v.z = __fmul_rn(v.z, scale);
      v.w = __fmul_rn(v.w, scale);
      const int64_t o4 = b4 + j;
      for (int r = 0; r < A.n; ++r)
        put4<OutT>(static_cast<char*>(peers.base[r]) + A.out_off, o4, v);
    }
  }
  HP_SPAN_END(SP_AR_RG);  // published by k_signal(1), next in the stream
}


// ---- copy-engine variant: the NVLink phases are cudaMemcpyAsync peer copies
// (no SMs), flags are raised by one-warp kernels after the copies complete in
// stream order; only the local source-order sum runs on the SMs.
// which 0: epoch + 1 -> push_flag[me] at every rank (and my epoch); which 1:
// epoch - lag -> applied_flag[me] (lag: buckets still to come this step).
__global__ void k_signal(void* my_win, PeerTable peers, int n, int me, int which, int lag) {
  HP_ENTRY(which ? SP_AR_WAIT1 : SP_AR_WAIT0);
  SigView sig(my_win);
  const int e = which == 0 ? *sig.epoch + 1 : *sig.epoch - lag;
  __threadfence_system();
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    SigView peer(peers.base[r]);
    st_release_sys(which == 0 ? &peer.push_flag[me] : &peer.applied_flag[me], e);
  }
  __syncwarp();
  if (which == 0 && threadIdx.x == 0) *sig.epoch = e;
  HP_SPAN_END(which ? SP_AR_WAIT1 : SP_AR_WAIT0);
}

// out[my chunk] = cast(scale * sum_s slot_s) in source-rank order; my own
// contribution is read straight from grad (zero past S_real).
template <typename OutT>
__global__ void __launch_bounds__(256)
k_ar_reduce_local(void* my_win, ArLayout A, const float4* __restrict__ grad, float scale) {
  HP_ENTRY(SP_AR_RG);
  const int64_t b4 = A.off4[A.me], c4 = A.off4[A.me + 1] - b4;
  const int64_t own_lim = min(c4, max((int64_t)0, (A.S_real >> 2) - b4));
  const float4* slots = reinterpret_cast<const float4*>(static_cast<char*>(my_win) + A.slots_off);
  const float4* mine = grad + b4;
  char* out = static_cast<char*>(my_win) + A.out_off;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < c4; j0 += 2 * stride) {
    float4 acc[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u * stride;
      acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < c4)
        for (int sidx = 0; sidx < A.n; ++sidx) {
          const float4 x = sidx == A.me ? (j < own_lim ? ldg_stream(mine + j)
                                                        : make_float4(0.f, 0.f, 0.f, 0.f))
                                        : ldg_stream(slots + (int64_t)sidx * A.sstride4 + j);
          acc[u] = f4_add(acc[u], x);
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u * stride;
      if (j >= c4) continue;
      float4 v = acc[u];
      v.x = __fmul_rn(v.x, scale);
      v.y = __fmul_rn(v.y, scale);
      v.z = __fmul_rn(v.z, scale);
      v.w = __fmul_rn(v.w, scale);
      put4<OutT>(out, b4 + j, v);
    }
  }
  HP_SPAN_END(SP_AR_RG);
}

// ---- one-shot pull variant (HP_DAR_PULL, the default at n = 2): every rank
// copies its gradient into its own window (slot [me]), publishes it, and then
// reads every peer's whole copy over NVLink and sums all n in rank order (own
// contribution from grad) -> scale -> cast -> its own output. One NVLink phase
// (each rank reads (n-1) S: at n = 2 the same bytes per direction as the two
// store phases, with one exchange of flags fewer and no second kernel on the
// peer's links); "applied" then tells each peer its copy may be overwritten by
// the next step (checked before the next copy).
__global__ void __launch_bounds__(256)
k_ar_copy_in(void* my_win, ArLayout A, const float4* __restrict__ grad) {
  HP_ENTRY(SP_AR_SCATTER);
  float4* in = reinterpret_cast<float4*>(static_cast<char*>(my_win) + A.slots_off) +
               (int64_t)A.me * A.sstride4;
  const int64_t n4 = A.S_real >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < n4; j0 += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < n4) v[u] = ldg_stream(grad + j);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < n4) in[j] = v[u];
    }
  }
  HP_SPAN_END(SP_AR_SCATTER);
}

template <typename OutT>
__global__ void __launch_bounds__(256)
k_ar_pull_sum(PeerTable peers, void* my_win, ArLayout A, const float4* __restrict__ grad, float scale) {
  HP_ENTRY(SP_AR_RG);
  const int64_t n4 = A.S_real >> 2, stride = (int64_t)gridDim.x * blockDim.x;
  char* out = static_cast<char*>(my_win) + A.out_off;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < n4; j0 += 2 * stride) {
    float4 x[2][AR_MAXN > 8 ? 8 : AR_MAXN];
    // issue every contribution's loads first (NVLink latency), then sum in rank order
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u * stride;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (s >= A.n || j >= n4) continue;
        x[u][s] = s == A.me ? ldg_stream(grad + j)
                            : reinterpret_cast<const float4*>(static_cast<const char*>(peers.base[s]) +
                                                              A.slots_off)[(int64_t)s * A.sstride4 + j];
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u * stride;
      if (j >= n4) continue;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < A.n) v = f4_add(v, x[u][s]);
      v.x = __fmul_rn(v.x, scale);
      v.y = __fmul_rn(v.y, scale);
      v.z = __fmul_rn(v.z, scale);
      v.w = __fmul_rn(v.w, scale);
      put4<OutT>(out, j, v);
    }
  }
  HP_SPAN_END(SP_AR_RG);
}

// ---- pipelined variant (HP_DAR_PIPE): ONE persistent kernel per rank. Every
// chunk is cut into pieces of AR_PIECE4 float4; the work items are, in queue
// order, (a) "scatter piece k of chunk c to rank c" for every peer c, then
// (b) "reduce piece k of my chunk". A block that finished storing a scatter
// piece raises the piece's arrival counter at its owner (system-scope atomic
// after a system fence); a reduce item waits for the n-1 arrivals of its piece,
// sums the n contributions in source-rank order (own contribution read from
// grad), scales, casts and stores the result into every rank's output. Items
// are taken from a device queue in order, so no block spins on a reduce item
// before every scatter item of its rank has been taken by a running block:
// no deadlock whatever the residency. The scatter of piece k+1 and the reduce
// of piece k overlap, so both NVLink directions carry both phases at once.
// Arrival counters are monotonic (epoch e expects e * (n-1)); the last block
// raises applied_flag[me] = e at every rank, resets the queue and bumps epoch.
constexpr int64_t AR_PIECE4 = 4096;  // 64 KB of fp32 per work item

template <typename OutT>
__global__ void __launch_bounds__(256)
k_ar_pipe(PeerTable peers, void* my_win, ArLayout A, const float4* __restrict__ grad, float scale,
          int* __restrict__ arrive, int* __restrict__ queue, long long timeout_cycles) {
  __shared__ int s_item;
  __shared__ bool s_last;
  HP_ENTRY(SP_AR_SCATTER);
  SigView sig(my_win);
  const int n = A.n, me = A.me;
  const int e = *sig.epoch + 1;
  const int64_t c4 = A.chunk >> 2, real4 = A.S_real >> 2;
  const int K = (int)((c4 + AR_PIECE4 - 1) / AR_PIECE4);
  const int n_sc = (n - 1) * K, n_items = n_sc + K;
  const float4* slots = reinterpret_cast<const float4*>(static_cast<char*>(my_win) + A.slots_off);
  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= n_items) break;
    if (it < n_sc) {  // scatter piece k of chunk c (the j-th peer after me) into rank c's slot [me]
      const int k = it / (n - 1), c = (me + 1 + it % (n - 1)) % n;
      const int64_t lo = (int64_t)k * AR_PIECE4, hi = min(c4, lo + AR_PIECE4);
      const int64_t lim = min(hi, max((int64_t)0, real4 - (int64_t)c * c4));
      const float4* src = grad + (int64_t)c * c4;
      float4* dst = reinterpret_cast<float4*>(static_cast<char*>(peers.base[c]) + A.slots_off) +
                    (int64_t)me * A.sstride4;
      for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += 4 * 256) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u * 256;
          v[u] = j < lim ? ldg_stream(src + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t j = j0 + u * 256;
          if (j < hi) dst[j] = v[u];
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        int* ctr = reinterpret_cast<int*>(static_cast<char*>(peers.base[c]) +
                                          (reinterpret_cast<char*>(arrive) - static_cast<char*>(my_win))) + k;
        asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
      }
    } else {  // reduce piece k of my chunk
      const int k = it - n_sc;
      if (threadIdx.x == 0 && n > 1) {
        const long long t0 = clock64();
        while (ld_acquire_sys(&arrive[k]) < e * (n - 1)) {
          if (clock64() - t0 > timeout_cycles) {
            atomicOr(sig.err, 4);
            break;
          }
          __nanosleep(32);
        }
      }
      __syncthreads();
      const int64_t lo = (int64_t)k * AR_PIECE4, hi = min(c4, lo + AR_PIECE4);
      const int64_t own_lim = min(c4, max((int64_t)0, real4 - (int64_t)me * c4));
      const float4* mine = grad + (int64_t)me * c4;
      for (int64_t j0 = lo + threadIdx.x; j0 < hi; j0 += 2 * 256) {
        float4 acc[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t j = j0 + u * 256;
          acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (j < hi)
            for (int s = 0; s < n; ++s) {
              const float4 x = s == me ? (j < own_lim ? ldg_stream(mine + j)
                                                      : make_float4(0.f, 0.f, 0.f, 0.f))
                                       : ldg_stream(slots + (int64_t)s * A.sstride4 + j);
              acc[u] = f4_add(acc[u], x);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t j = j0 + u * 256;
          if (j >= hi) continue;
          float4 v = acc[u];
          v.x = __fmul_rn(v.x, scale);
          v.y = __fmul_rn(v.y, scale);
          v.z = __fmul_rn(v.z, scale);
          v.w = __fmul_rn(v.w, scale);
          const int64_t o4 = (int64_t)me * c4 + j;
          for (int r = 0; r < n; ++r) {
            const int d = (me + 1 + r) % n;  // peers first, own output last
            put4<OutT>(static_cast<char*>(peers.base[d]) + A.out_off, o4, v);
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    __threadfence_system();
    s_last = atomicAdd(&sig.done[3], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence_system();
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      st_release_sys(&SigView(peers.base[r]).applied_flag[me], e);
    __syncthreads();
    if (threadIdx.x == 0) {
      *sig.epoch = e;
      *queue = 0;
      sig.done[3] = 0;
    }
  }
  HP_SPAN_END(SP_AR_SCATTER);
}

}  // namespace
}  // namespace hp

struct hp_dar_s {
  ArLayout A;
  void* win;
  PeerTable peers;
  int64_t arrive_off, queue_off;  // HP_DAR_PIPE: piece arrival counters, work queue
  bool weighted;                  // hp_dar_set_split gave a non-uniform split
  uint64_t ipc_mask;              // peers mapped with cudaIpcOpenMemHandle
  int mode;                  // HP_DAR_SM | HP_DAR_CE | HP_DAR_PIPE
  cudaStream_t side[4];      // CE mode: copies to different peers run concurrently
  cudaEvent_t fork, join[4];
  bool side_ready;           // side streams / events created (CE mode only)
};

// CE mode's side streams, created once on first use (SM / pipelined modes never
// hold extra streams: fewer streams per rank share the device's hardware queues)
static int dar_side_streams(hp_dar_s* d) {
  if (d->side_ready) return HP_OK;
  for (int k = 0; k < 4; ++k) {
    HP_CUDA(cudaStreamCreateWithFlags(&d->side[k], cudaStreamNonBlocking));
    HP_CUDA(cudaEventCreateWithFlags(&d->join[k], cudaEventDisableTiming));
  }
  HP_CUDA(cudaEventCreateWithFlags(&d->fork, cudaEventDisableTiming));
  d->side_ready = true;
  return HP_OK;
}

extern "C" {

// Symmetric window of one dense Weight: [sig][slots n x chunk fp32][out S].
// S (elements, a multiple of 4) is padded internally to a multiple of 4 * n.
// Returns the cudaIpc handle and the output pointer (out_dtype = HP_DTYPE_F32
// or HP_DTYPE_BF16; the first S elements are the result).
int hp_dar_create(hp_dar_t* out, int32_t n, int32_t me, int64_t S_real, int32_t out_dtype,
                  void* ipc_handle_out, void** out_ptr) {
  HP_REQUIRE(out && ipc_handle_out && out_ptr && n >= 1 && n <= AR_MAXN && me >= 0 && me < n,
             "bad dense allreduce args");
  HP_REQUIRE(S_real > 0 && S_real % 4 == 0, "S must be a positive multiple of 4");
  const int64_t S = (S_real + 4 * n - 1) / (4 * n) * (4 * n);
  HP_REQUIRE(out_dtype == HP_DTYPE_F32 || out_dtype == HP_DTYPE_BF16, "out dtype f32 | bf16");
  auto* d = new hp_dar_s{};
  auto al = [](int64_t v) { return (v + 255) & ~(int64_t)255; };
  d->A.S = S;
  d->A.S_real = S_real;
  d->A.n = n;
  d->A.me = me;
  d->A.chunk = S / n;
  d->A.out_bytes = out_dtype == HP_DTYPE_F32 ? 4 : 2;
  d->A.in_bytes = 4;
  // slots sized for any split (a chunk may be all of S): n sources x S
  d->A.sstride4 = S / 4;
  for (int r = 0; r <= n; ++r) d->A.off4[r] = (int64_t)r * (S / n) / 4;
  d->A.slots_off = al(SIG_INTS * 4);
  d->A.out_off = d->A.slots_off + al((int64_t)n * S * 4);
  d->arrive_off = d->A.out_off + al(S * d->A.out_bytes);
  d->queue_off = d->arrive_off + al(((S / n / 4 + AR_PIECE4 - 1) / AR_PIECE4) * 4);
  const int64_t bytes = d->queue_off + 256;
  cudaError_t e = cudaMalloc(&d->win, bytes);
  if (e != cudaSuccess) {
    delete d;
    return cuda_fail(e, "cudaMalloc(dense window)");
  }
  HP_CUDA(cudaMemset(d->win, 0, bytes));  // slot padding must read as zeros
  d->mode = HP_DAR_CE;  // side streams for the copies: created on first CE use
  cudaIpcMemHandle_t h;
  HP_CUDA(cudaIpcGetMemHandle(&h, d->win));
  memcpy(ipc_handle_out, &h, sizeof(h));
  for (int r = 0; r < 64; ++r) d->peers.base[r] = nullptr;
  d->peers.base[me] = d->win;
  *out_ptr = static_cast<char*>(d->win) + d->A.out_off;
  *out = d;
  return HP_OK;
}

int hp_dar_open_peer(hp_dar_t d, int32_t rank, const void* ipc_handle) {
  HP_REQUIRE(d && rank >= 0 && rank < d->A.n && ipc_handle, "bad peer args");
  if (rank == d->A.me) return HP_OK;
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  void* p = nullptr;
  HP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  d->peers.base[rank] = p;
  d->ipc_mask |= 1ull << rank;
  return HP_OK;
}

// Single-process emulation (see hp_xchg_set_peer_ptr).
int hp_dar_window_ptr(hp_dar_t d, void** out) {
  HP_REQUIRE(d && out, "NULL argument");
  *out = d->win;
  return HP_OK;
}

int hp_dar_set_peer_ptr(hp_dar_t d, int32_t rank, void* window) {
  HP_REQUIRE(d && rank >= 0 && rank < d->A.n && window, "bad peer args");
  if (rank == d->A.me) return HP_OK;
  HP_REQUIRE(!((d->ipc_mask >> rank) & 1ull), "peer already mapped by IPC");
  d->peers.base[rank] = window;
  return HP_OK;
}

int hp_dar_destroy(hp_dar_t d) {
  if (!d) return HP_OK;
  for (int r = 0; r < d->A.n; ++r)
    if (r != d->A.me && ((d->ipc_mask >> r) & 1ull)) cudaIpcCloseMemHandle(d->peers.base[r]);
  if (d->side_ready) {
    for (int k = 0; k < 4; ++k) {
      cudaStreamDestroy(d->side[k]);
      cudaEventDestroy(d->join[k]);
    }
    cudaEventDestroy(d->fork);
  }
  cudaFree(d->win);
  delete d;
  return HP_OK;
}

// out (the window's output, every rank) = cast(scale * sum_r grad_r), summed in
// rank order. grad is this rank's fp32 gradient [S] (any device buffer).
// Chunk split of the reduction: rank r reduces (and gathers) a share of S
// proportional to weights[r] >= 0 (rounded to float4; identical weights on
// every rank). A rank with weight 0 only scatters its gradient and receives the
// result: its NVLink egress drops from 2(n-1)/n S to S - its chunk = S, which
// relieves a rank whose links also carry a hot sparse partition.
int hp_dar_set_split(hp_dar_t d, const double* weights) {
  HP_REQUIRE(d && weights, "NULL argument");
  const int n = d->A.n;
  double tot = 0;
  for (int r = 0; r < n; ++r) {
    HP_REQUIRE(weights[r] >= 0, "weights must be >= 0");
    tot += weights[r];
  }
  HP_REQUIRE(tot > 0, "at least one weight must be > 0");
  const int64_t S4 = d->A.S / 4;
  double acc = 0;
  bool uniform = true;
  for (int r = 0; r < n; ++r) {
    d->A.off4[r] = (int64_t)(acc / tot * (double)S4 + 0.5);
    acc += weights[r];
    uniform = uniform && weights[r] == weights[0];
  }
  d->A.off4[n] = S4;
  if (uniform)
    for (int r = 0; r <= n; ++r) d->A.off4[r] = (int64_t)r * (d->A.S / n) / 4;
  d->weighted = !uniform;
  return HP_OK;
}

int hp_dar_set_mode(hp_dar_t d, int32_t mode) {
  HP_REQUIRE(d && (mode == HP_DAR_SM || mode == HP_DAR_CE || mode == HP_DAR_PIPE ||
                  mode == HP_DAR_PULL),
             "mode must be HP_DAR_SM, HP_DAR_CE, HP_DAR_PIPE or HP_DAR_PULL");
  HP_REQUIRE(mode != HP_DAR_PULL || d->A.n <= 8, "the pull exchange sums at most 8 ranks");
  d->mode = mode;
  return mode == HP_DAR_CE ? dar_side_streams(d) : HP_OK;
}

// CE mode: chunk copies to every peer, fanned out over the side streams.
static int dar_copies(hp_dar_t d, cudaStream_t st, bool gather, const float* grad) {
  if (int rc = dar_side_streams(d)) return rc;
  const ArLayout& A = d->A;
  const int npeer = A.n - 1;
  const int ns = npeer < 4 ? npeer : 4;
  HP_CUDA(cudaEventRecord(d->fork, st));
  for (int k = 0; k < ns; ++k) HP_CUDA(cudaStreamWaitEvent(d->side[k], d->fork, 0));
  int q = 0;
  for (int r = 0; r < A.n; ++r) {
    if (r == A.me) continue;
    cudaStream_t cs = d->side[q++ % ns];
    if (!gather) {  // my chunk r -> rank r's slot [me]
      const int64_t b = A.off4[r] * 4, len = A.off4[r + 1] * 4 - b;
      const int64_t real = std::min(len, std::max((int64_t)0, A.S_real - b));
      if (real > 0)
        HP_CUDA(cudaMemcpyAsync(static_cast<char*>(d->peers.base[r]) + A.slots_off +
                                    (int64_t)A.me * A.sstride4 * 16,
                                grad + b, real * 4, cudaMemcpyDeviceToDevice, cs));
    } else {  // my reduced chunk -> rank r's output
      const int64_t b = A.off4[A.me] * 4, len = A.off4[A.me + 1] * 4 - b;
      const int64_t off = A.out_off + b * A.out_bytes;
      if (len > 0)
        HP_CUDA(cudaMemcpyAsync(static_cast<char*>(d->peers.base[r]) + off,
                                static_cast<char*>(d->win) + off, len * A.out_bytes,
                                cudaMemcpyDeviceToDevice, cs));
    }
  }
  for (int k = 0; k < ns; ++k) {
    HP_CUDA(cudaEventRecord(d->join[k], d->side[k]));
    HP_CUDA(cudaStreamWaitEvent(st, d->join[k], 0));
  }
  return HP_OK;
}

int hp_dar_allreduce(hp_dar_t d, const void* grad_v, float scale, void* stream) {
  HP_REQUIRE(d && grad_v && ((uintptr_t)grad_v & 15) == 0, "grad must be a 16-byte aligned buffer");
  HP_REQUIRE(d->A.in_bytes == 4 || d->mode == HP_DAR_SM,
             "bf16 gradients need the SM-store dense exchange (HP_DAR_SM)");
  const float* grad = static_cast<const float*>(grad_v);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int sms = sm_count();
  int64_t maxc = 0, myc = (d->A.off4[d->A.me + 1] - d->A.off4[d->A.me]) * 4;
  for (int r = 0; r < d->A.n; ++r) maxc = std::max(maxc, (d->A.off4[r + 1] - d->A.off4[r]) * 4);
  if (d->mode == HP_DAR_CE) {
    int rc;
    if (d->A.n > 1 && (rc = dar_copies(d, st, false, grad))) return rc;
    launch_k(k_signal, dim3(1), dim3(32), 0, st, d->win, d->peers, d->A.n, d->A.me, 0, 0);
    launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 0, d->A.n, wait_budget(), SP_AR_WAIT0, 0);
    const int brg = grid_for(myc / 8, 256, sms * 2);
    if (d->A.out_bytes == 4)
      launch_k(k_ar_reduce_local<float>, dim3(brg), dim3(256), 0, st, d->win, d->A,
               reinterpret_cast<const float4*>(grad), scale);
    else
      launch_k(k_ar_reduce_local<__nv_bfloat16>, dim3(brg), dim3(256), 0, st, d->win, d->A,
               reinterpret_cast<const float4*>(grad), scale);
    if (d->A.n > 1 && (rc = dar_copies(d, st, true, grad))) return rc;
    launch_k(k_signal, dim3(1), dim3(32), 0, st, d->win, d->peers, d->A.n, d->A.me, 1, 0);
    launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 1, d->A.n, wait_budget(), SP_AR_WAIT1, 0);
    HP_LAUNCHED(5, "dense p2p allreduce (copy engines)");
    return HP_OK;
  }
  if (d->mode == HP_DAR_PULL) {
    // the peers finished reading my previous copy (their "applied" of my epoch)
    launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 1, d->A.n, wait_budget(), SP_AR_WAIT1, 0);
    const int bc = grid_for(d->A.S_real / 16, 256, sms * 4);
    launch_k(k_ar_copy_in, dim3(bc), dim3(256), 0, st, d->win, d->A, reinterpret_cast<const float4*>(grad));
    launch_k(k_signal, dim3(1), dim3(32), 0, st, d->win, d->peers, d->A.n, d->A.me, 0, 0);
    launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 0, d->A.n, wait_budget(), SP_AR_WAIT0, 0);
    const int bp = grid_for(d->A.S_real / 8, 256, sms * 4);
    if (d->A.out_bytes == 4)
      launch_k(k_ar_pull_sum<float>, dim3(bp), dim3(256), 0, st, d->peers, d->win, d->A,
               reinterpret_cast<const float4*>(grad), scale);
    else
      launch_k(k_ar_pull_sum<__nv_bfloat16>, dim3(bp), dim3(256), 0, st, d->peers, d->win, d->A,
               reinterpret_cast<const float4*>(grad), scale);
    launch_k(k_signal, dim3(1), dim3(32), 0, st, d->win, d->peers, d->A.n, d->A.me, 1, 0);
    HP_LAUNCHED(6, "dense p2p allreduce (one-shot pull)");
    return HP_OK;
  }
  if (d->mode == HP_DAR_PIPE) {
    HP_REQUIRE(!d->weighted, "the pipelined dense exchange needs the uniform split");
    const int64_t c4 = d->A.chunk / 4;
    const int K = (int)((c4 + AR_PIECE4 - 1) / AR_PIECE4);
    const int blocks = std::max(1, std::min(d->A.n * K, g_dar_blocks > 0 ? g_dar_blocks : sms));
    int* arrive = reinterpret_cast<int*>(static_cast<char*>(d->win) + d->arrive_off);
    int* queue = reinterpret_cast<int*>(static_cast<char*>(d->win) + d->queue_off);
    if (d->A.out_bytes == 4)
      launch_k(k_ar_pipe<float>, dim3(blocks), dim3(256), 0, st, d->peers, d->win, d->A,
               reinterpret_cast<const float4*>(grad), scale, arrive, queue, wait_budget());
    else
      launch_k(k_ar_pipe<__nv_bfloat16>, dim3(blocks), dim3(256), 0, st, d->peers, d->win, d->A,
               reinterpret_cast<const float4*>(grad), scale, arrive, queue, wait_budget());
    launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 1, d->A.n, wait_budget(), SP_AR_WAIT1, 0);
    HP_LAUNCHED(2, "dense p2p allreduce (pipelined)");
    return HP_OK;
  }
  // SM stores in nb buckets (hp_debug_set_dar_buckets; default 1): every
  // chunk is cut into nb pieces; all scatters go first (each published with
  // its own epoch), then per bucket wait -> reduce/gather -> publish, so one
  // bucket's cross-GPU wait overlaps the other buckets' link traffic and only
  // the last gather's wait is exposed. Epochs advance by nb per step.
  // Measured at N = 2 (LM1B dense): every extra bucket costs ~17 us of kernel
  // boundaries (5 more dependent launches) for ~6 us of hidden wait, so 1.
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(g_dar_buckets, std::max<int64_t>(1, maxc / 4096)));
  // scatter grid: ~half the SMs (the sparse tables' kernels run beside it);
  // hp_debug_set_dar_blocks / _dar_rg_blocks (b > 0): b blocks in total per
  // scatter / per reduce-gather (A/B)
  const int np = d->A.n - 1;
  const int bx = g_dar_blocks > 0 ? std::max(1, g_dar_blocks / std::max(1, np))
                                  : std::max(1, std::min(grid_for(maxc / nb / 16, 256, sms),
                                                         sms / std::max(1, np)));
  const int brg = g_dar_rg_blocks > 0 ? g_dar_rg_blocks
                                      : grid_for(std::max<int64_t>(myc / nb, 8) / 8, 256, sms * 2);
  const void* g = grad;
  const bool bf_in = d->A.in_bytes == 2;
  for (int b = 0; b < nb; ++b) {
    if (np > 0) {
      if (bf_in)
        launch_k(k_ar_scatter<__nv_bfloat16>, dim3(bx, np), dim3(256), 0, st, d->peers, d->A, g, b, nb);
      else if (g_dar_tma) {  // A/B: TMA bulk copies, g_dar_tma CTAs per peer chunk
        static bool tconf = false;
        if (!tconf) {
          HP_CUDA(cudaFuncSetAttribute(k_ar_scatter_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       2 * AR_TMA_F4 * 16));
          tconf = true;
        }
        launch_k(k_ar_scatter_tma, dim3(g_dar_tma, np), dim3(32), 2 * AR_TMA_F4 * 16, st, d->peers,
                 d->A, static_cast<const float4*>(g));
      } else if (g_dar_deep)  // A/B: 16 vectors in flight per thread (fewer CTAs saturate the link)
        launch_k(k_ar_scatter<float, 16>, dim3(bx, np), dim3(256), 0, st, d->peers, d->A, g, b, nb);
      else
        launch_k(k_ar_scatter<float>, dim3(bx, np), dim3(256), 0, st, d->peers, d->A, g, b, nb);
    }
    launch_k(k_signal, dim3(1), dim3(32), 0, st, d->win, d->peers, d->A.n, d->A.me, 0, 0);
  }
  for (int b = 0; b < nb; ++b) {
    const int lag = nb - 1 - b;
    launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 0, d->A.n, wait_budget(), SP_AR_WAIT0, lag);
    const dim3 G(brg), Bk(256);
    if (d->A.out_bytes == 4 && !bf_in && g_dar_rg_tma > 0 && nb == 1) {  // TMA reduce/gather
      static bool rconf = false;
      if (!rconf) {
        HP_CUDA(cudaFuncSetAttribute(k_ar_rg_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     3 * AR_RG_F4 * 16));
        rconf = true;
      }
      launch_k(k_ar_rg_tma, dim3(g_dar_rg_tma), dim3(128), 3 * AR_RG_F4 * 16, st, d->peers, d->win,
               d->A, static_cast<const float4*>(g), scale);
    } else if (d->A.out_bytes == 4 && !bf_in && g_dar_deep)
      launch_k(k_ar_reduce_gather<float, float, 8>, G, Bk, 0, st, d->peers, d->win, d->A, g, scale, b,
               nb);
    else if (d->A.out_bytes == 4 && !bf_in)
      launch_k(k_ar_reduce_gather<float, float>, G, Bk, 0, st, d->peers, d->win, d->A, g, scale, b, nb);
    else if (d->A.out_bytes == 4)
      launch_k(k_ar_reduce_gather<float, __nv_bfloat16>, G, Bk, 0, st, d->peers, d->win, d->A, g,
               scale, b, nb);
    else if (!bf_in)
      launch_k(k_ar_reduce_gather<__nv_bfloat16, float>, G, Bk, 0, st, d->peers, d->win, d->A, g,
               scale, b, nb);
    else
      launch_k(k_ar_reduce_gather<__nv_bfloat16, __nv_bfloat16>, G, Bk, 0, st, d->peers, d->win,
               d->A, g, scale, b, nb);
    launch_k(k_signal, dim3(1), dim3(32), 0, st, d->win, d->peers, d->A.n, d->A.me, 1, lag);
  }
  launch_k(k_wait, dim3(1), dim3(64), 0, st, d->win, 1, d->A.n, wait_budget(), SP_AR_WAIT1, 0);
  HP_LAUNCHED(nb * ((np > 0 ? 1 : 0) + 4) + 1, "dense p2p allreduce");
  return HP_OK;
}

int hp_dar_set_in_dtype(hp_dar_t d, int32_t in_dtype) {
  HP_REQUIRE(d && (in_dtype == HP_DTYPE_F32 || in_dtype == HP_DTYPE_BF16), "in dtype f32 | bf16");
  d->A.in_bytes = in_dtype == HP_DTYPE_F32 ? 4 : 2;
  return HP_OK;
}

int hp_dar_err_ptr(hp_dar_t d, const int32_t** out) {
  HP_REQUIRE(d && out, "NULL argument");
  *out = SigView(d->win).err;
  return HP_OK;
}

int hp_dar_status(hp_dar_t d, int32_t* out_err, void* stream) {
  HP_REQUIRE(d && out_err, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SigView sig(d->win);
  HP_CUDA(cudaMemcpyAsync(out_err, sig.err, 4, cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  return HP_OK;
}

}  // extern "C"

// ---- instrumentation: raw peer-memory throughput between this rank and
// rank `peer` over the dense window's slot region (bytes = S * 4).
namespace hp {
namespace {
template <int U, bool LOAD>
__global__ void __launch_bounds__(256) k_nvl_bench(float4* local, float4* remote, int64_t n4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n4) v[u] = LOAD ? remote[i] : local[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n4) {
        if (LOAD) acc = f4_add(acc, v[u]);
        else remote[i] = v[u];
      }
    }
  }
  if (LOAD && acc.x == 12345.f) local[0] = acc;  // keep the loads
}
}  // namespace
}  // namespace hp

// ---- instrumentation: cost of the per-block publication pattern. Every block
// stores `per_block` float4 to the peer (0 = none), then: mode 0 nothing,
// 1 __syncthreads + thread 0 fence.sc.sys, 2 fence.sc.gpu, 3 fence.acq_rel.sys.
namespace hp {
namespace {
__global__ void k_fence_bench(float4* remote, int per_block, int mode, int* ctr) {
  float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  float4* dst = remote + (int64_t)blockIdx.x * per_block;
  for (int i = threadIdx.x; i < per_block; i += blockDim.x) dst[i] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 1) __threadfence_system();
    else if (mode == 2) __threadfence();
    else if (mode == 3) asm volatile("fence.acq_rel.sys;" ::: "memory");
    atomicAdd(ctr, 1);
  }
}
}  // namespace
}  // namespace hp

extern "C" int hp_debug_fence_bench(hp_dar_t d, int32_t peer, int32_t mode, int32_t blocks,
                                    int32_t per_block, void* stream) {
  HP_REQUIRE(d && peer >= 0 && peer < d->A.n && d->peers.base[peer], "bad peer");
  HP_REQUIRE((int64_t)blocks * per_block <= d->A.S / 4, "fence bench exceeds the slot region");
  float4* remote = reinterpret_cast<float4*>(static_cast<char*>(d->peers.base[peer]) + d->A.slots_off);
  int* ctr = reinterpret_cast<int*>(static_cast<char*>(d->win) + d->queue_off) + 8;
  k_fence_bench<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(remote, per_block, mode, ctr);
  HP_CUDA(cudaGetLastError());
  return HP_OK;
}

extern "C" int hp_debug_nvlink_bench(hp_dar_t d, int32_t peer, int32_t mode, int32_t blocks,
                                     void* stream) {
  HP_REQUIRE(d && peer >= 0 && peer < d->A.n && d->peers.base[peer], "bad peer");
  float4* local = reinterpret_cast<float4*>(static_cast<char*>(d->win) + d->A.slots_off);
  float4* remote = reinterpret_cast<float4*>(static_cast<char*>(d->peers.base[peer]) + d->A.slots_off);
  const int64_t n4 = d->A.S / 4;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (mode) {
    case 0: k_nvl_bench<1, false><<<blocks, 256, 0, st>>>(local, remote, n4); break;
    case 1: k_nvl_bench<1, true><<<blocks, 256, 0, st>>>(local, remote, n4); break;
    case 2: k_nvl_bench<4, false><<<blocks, 256, 0, st>>>(local, remote, n4); break;
    default: k_nvl_bench<4, true><<<blocks, 256, 0, st>>>(local, remote, n4); break;
  }
  HP_CUDA(cudaGetLastError());
  return HP_OK;
}
