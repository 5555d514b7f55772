// K1 + K2: on-device radix sort of row ids, segment (dedup) metadata and
// partition routing. Produces the DedupPlan the reduce/apply kernels consume.
//
// Reference semantics replaced: local aggregation ("iterating through nonzero
// indices one by one to accumulate values with the same index", PAPER.md:471;
// placement.py:155-161) and routing (model.py:36-44, 192-204; placement.py:95-97,
// 185-193). Output order and the summation tree are specified in oracle/oracle.py.
//
// Two paths:
//  * T <= HP_SMALL_MAX: ONE CTA sorts in shared memory (warp-striped items,
//    __match_any_sync multisplit ranking, 8-bit digits) and derives every index
//    structure in the same launch (LM/NMT shapes: 2.5k-11k ids per table).
//  * larger T: LSD radix sort over 4096-key tiles (tile histogram -> per-digit
//    column scan -> stable in-tile rank + smem-staged coalesced scatter), then
//    grid-wide metadata kernels with a reduce-then-scan device scan.
#include <cooperative_groups.h>

#include "hp_dedup.cuh"

namespace hp {

namespace {

constexpr int HS = HP_RADIX + 1;  // padded histogram row (bank spread)

// Sort key of position i. An id outside [0, V) is DROPPED, never clamped onto a
// real row: its key becomes the sentinel V (key_bits holds V, so it sorts after
// every row), its segment gets no send slot and destination -1 (the reduce
// skips it), inv = -1 (stitch writes a zero row), and error bit 1 is raised
// for the runner. TF1's SparseApply* rejects such indices the same way.
__device__ __forceinline__ uint32_t load_key(const int64_t* ids, int64_t i, int64_t V, int* err) {
  int64_t id = ids[i];
  if (id < 0 || id >= V) {
    if (err) atomicOr(err, 1);
    id = V;
  }
  return (uint32_t)id;
}

// Stable rank of NT*IPT warp-striped items by an 8-bit digit.
// Item (warp w, round r, lane l) has tile index w*32*IPT + r*32 + l; ranks
// preserve that order within a digit. s_hist: NW*HS ints, s_scan: 33 ints.
// On return s_hist[d] (warp 0 row) = first rank of digit d in the tile.
template <int NT, int IPT>
__device__ __forceinline__ void block_rank(const uint32_t (&key)[IPT], int shift, int (&rank)[IPT],
                                           int* s_hist, int* s_scan) {
  constexpr int NW = NT / 32;
  constexpr int E = NW * HP_RADIX;
  constexpr int PER = E / NT;
  static_assert(E % NT == 0, "histogram must split evenly");
  const int w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NW * HS; i += NT) s_hist[i] = 0;
  __syncthreads();
  int* my = s_hist + w * HS;
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const unsigned d = (key[r] >> shift) & (HP_RADIX - 1);
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int before = __popc(peers & lt);
    const int cnt = my[d];
    rank[r] = cnt + before;
    __syncwarp();
    if (before == 0) my[d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // Exclusive scan over (digit, warp) in digit-major order.
  int v[PER];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x * PER + k;
    v[k] = s_hist[(e % NW) * HS + e / NW];
    sum += v[k];
  }
  int total;
  int base = block_excl_scan<NT>(sum, s_scan, &total);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x * PER + k;
    s_hist[(e % NW) * HS + e / NW] = base;
    base += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < IPT; ++r) rank[r] += my[(key[r] >> shift) & (HP_RADIX - 1)];
}

// Owner-grouped send-slot bases: part_base[p] = dest_off[owner[p]] +
// sum_{p'<p, owner[p']==owner[p]} cnt[p']. Runs inside ONE block of NT threads.
template <int NT>
__device__ void partition_bases(const int32_t* first_u, const int32_t* owner, int P, int nranks,
                                int32_t* part_base, int32_t* dest_counts, int* s_dest) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = w; o < nranks; o += NW) {
    int carry = 0;
    for (int pb = 0; pb < P; pb += 32) {
      const int p = pb + lane;
      const bool mine = p < P && (owner ? owner[p] : 0) == o;
      const int c = mine ? first_u[p + 1] - first_u[p] : 0;
      const int incl = warp_incl_scan(c);
      if (mine) part_base[p] = carry + incl - c;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      s_dest[o] = carry;
      if (dest_counts) dest_counts[o] = carry;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int o = 0; o < nranks; ++o) {
      const int c = s_dest[o];
      s_dest[o] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += NT) part_base[p] += s_dest[owner ? owner[p] : 0];
  __syncthreads();
}

__device__ __forceinline__ int lower_bound_u32(const uint32_t* a, int n, uint32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

constexpr int MAX_RANKS = 1024;

// Destination row of a segment: its send slot (send plans) or its row in the
// caller's slab (apply plans; -1 + error bit if the row is not homed here).
__device__ __forceinline__ int seg_dst(uint32_t id, int p, int slot, const int64_t* dst_pb,
                                       const Router& route, int* err) {
  if (!dst_pb) return slot;
  const int64_t b = dst_pb[p];
  if (b < 0) {
    atomicOr(err, 2);
    return -1;
  }
  return (int)(b + ((int64_t)id - route.lo(p)));
}

// Reduce items of segment u: chunks of HP_CHUNK sorted rows. Short segments
// (one chunk) are final and write straight to dst; long ones write partial
// slots bp.. and get a long descriptor for k_combine.
// A single-row segment (the common case) carries its row's original position
// directly: item.x = -(pos + 1), saving the reduce kernel one dependent load.
// Item `it` covers sorted rows [r, r+n): record it as the first item of every
// row-stream warp whose row cut w*R falls at its start, and the next item for
// cuts inside it.
__device__ __forceinline__ void emit_bounds(const DedupPlan& pl, int it, int r, int n) {
  if (pl.nw <= 0) return;
  const int T = (int)pl.T;
  const int R = (T + pl.nw - 1) / pl.nw;
  for (int w = (r + R - 1) / R; (int64_t)w * R < r + n; ++w) {
    const bool at = w * R == r;
    pl.wb_item[w] = at ? it : it + 1;
    pl.wb_row[w] = at ? r : r + n;
  }
}

// Item order (no row stream, pl.nw == 0): the chunks of every long segment
// come FIRST, at item index = their partial slot (bp + k), so the hot ids'
// chunks run in k_reduce's first wave and the fused upper levels of their
// trees (combine_up, the last arriver of each group) finish early instead of
// in a separate k_combine at the tail. Long chunks carry w = -(long index + 1);
// short items (w = 1) follow at tot_p + (short items before). Without the
// fused tree (pl.fused == 0) items stay in sorted-row order (long chunks not final,
// k_combine runs the upper levels). Every long chunk carries its segment's
// long index (w = -(li+1)): the stitch (k_bcast_rows) finds the segment's row.
__device__ __forceinline__ void emit_items(const DedupPlan& pl, int u, int j0, int L, int dst,
                                           int bi, int bp, int bl, int pos0, int tot_p) {
  const int n0 = (L + HP_CHUNK - 1) / HP_CHUNK;
  const bool lg = L > HP_CHUNK;
  const bool reorder = pl.reorder != 0;
  const int si = reorder ? tot_p + (bi - bp) : bi;  // index of a short segment's item
  if (L == 1) {
    pl.items[si] = make_int4(-(pos0 + 1), 1, dst, 1);
    emit_bounds(pl, bi, j0, 1);
    return;
  }
  for (int k = 0; k < n0; ++k) {
    const int n = min(HP_CHUNK, L - k * HP_CHUNK);
    const int idx = !lg ? si + k : (reorder ? bp + k : bi + k);
    pl.items[idx] = make_int4(j0 + k * HP_CHUNK, n, lg ? bp + k : dst, lg ? -(bl + 1) : 1);
    if (lg) pl.part_desc[bp + k] = make_int4(j0 + k * HP_CHUNK, n, dst, bl);
    emit_bounds(pl, bi + k, j0 + k * HP_CHUNK, n);
  }
  if (lg) {
    pl.longs[bl] = make_int4(bp, n0, dst, L);  // {partial slot, chunks, dst, rows}
    pl.long_flag[bl] = 0;
  }
}

// ------------------------------------------------------------------ cluster path
// T <= HP_SMALL_MAX: one thread-block cluster of CS CTAs sorts the ids in
// distributed shared memory. CTA c owns sorted slice [c*S, (c+1)*S); each LSD
// pass ranks the slice locally (warp multisplit), publishes its digit counts,
// and after a cluster barrier scatters every (key, pos) straight into the
// owning CTA's shared memory (DSMEM stores).
// Metadata needs ONE more barrier: each CTA analyses the segments whose head
// lies in its slice (lengths, reduce items, per-partition unique counts) from
// shared memory, publishes a few scalars and its partition histogram, and after
// the barrier derives every global offset it needs (segment / item / partial
// prefixes, partition bases) from the other CTAs' published state.
constexpr int CL_PMAX = 2048;  // partitions handled by the cluster path

// Published per-CTA scalars (s_pub).
enum { PB_HEADS = 0, PB_FIRST, PB_LAST, PB_ITEMS, PB_PARTS, PB_LONGS, PB_N };

__device__ __forceinline__ int pack3(int a, int b, int c) { return a | (b << 12) | (c << 22); }

template <int NT, int IPT, int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(NT, 1)
k_dedup_cluster(DedupPlan pl, const int64_t* __restrict__ ids, const int32_t* __restrict__ owner,
                const int64_t* __restrict__ dst_pb, int64_t* send_ids, int32_t* counts,
                int32_t* inv, int32_t* dest_counts, int32_t* n_uniq) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int S = NT * IPT, NW = NT / 32;
  static_assert(S < 4096, "packed scan fields are 12/10/10 bits");
  extern __shared__ __align__(16) unsigned char smem[];
  uint2* s_buf = reinterpret_cast<uint2*>(smem);  // sorted slice (key, pos)
  int* s_hist = reinterpret_cast<int*>(s_buf + S);
  int* s_hpos = s_hist + NW * HS;  // local head positions [S]
  int* s_sig = s_hpos + S;         // send slot of local segment [S]
  int* s_scan = s_sig + S;
  int* s_cnt = s_scan + 40;      // published digit counts
  int* s_base = s_cnt + HP_RADIX;
  int* s_pub = s_base + HP_RADIX;  // published scalars
  int* s_dest = s_pub + 16;
  int* s_pcnt = s_dest + MAX_RANKS;  // published unique counts per partition
  int* s_first = s_pcnt + CL_PMAX;   // first unique index of partition p (P+1)
  int* s_pbase = s_first + CL_PMAX + 1;
  const int c = (int)cl.block_rank();
  const int T = (int)pl.T, P = pl.P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const Router route(pl.V, P);
  HP_ENTRY(SP_DEDUP);
  int nprof = 0;
#define HP_PROF()                                                     \
  do {                                                                \
    if (pl.prof && tid == 0) pl.prof[c * 16 + nprof] = clock64();     \
    ++nprof;                                                          \
  } while (0)
  HP_PROF();
  // Error bits gather in shared memory and reach counters[C_ERR] once per CTA
  // at the end; CTA 0 zeroes the word first (ordered by the cluster barriers
  // in between), so the plan needs no memset node in front of this kernel.
  __shared__ int s_err;
  if (tid == 0) {
    s_err = 0;
    if (c == 0) {
      pl.counters[C_ERR] = 0;
      pl.counters[C_QUEUE] = 0;
      pl.counters[C_DONE] = 0;
      pl.counters[C_GEN] = 0;
    }
  }
  __syncthreads();

  uint32_t key[IPT];
  int32_t pos[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int i = c * S + w * 32 * IPT + r * 32 + lane;
    key[r] = i < T ? load_key(ids, i, pl.V, &s_err) : 0xffffffffu;
    pos[r] = i;
  }
  HP_PROF();
  const int passes = (pl.key_bits + HP_RADIX_BITS - 1) / HP_RADIX_BITS;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * HP_RADIX_BITS;
    int rank[IPT];
    block_rank<NT, IPT>(key, shift, rank, s_hist, s_scan);
    if (tid < HP_RADIX) s_cnt[tid] = (tid + 1 < HP_RADIX ? s_hist[tid + 1] : S) - s_hist[tid];
    HP_PROF();
    cl.sync();
    int tot = 0, pre = 0;
    if (tid < HP_RADIX) {
#pragma unroll
      for (int cc = 0; cc < CS; ++cc) {
        const int v = cl.map_shared_rank(s_cnt, cc)[tid];
        tot += v;
        pre += cc < c ? v : 0;
      }
    }
    int all;
    const int ex = block_excl_scan<NT>(tid < HP_RADIX ? tot : 0, s_scan, &all);
    if (tid < HP_RADIX) s_base[tid] = ex + pre - s_hist[tid];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < IPT; ++r) {
      const int g = s_base[(key[r] >> shift) & (HP_RADIX - 1)] + rank[r];
      const int dc = g / S;
      cl.map_shared_rank(s_buf, dc)[g - dc * S] = make_uint2(key[r], (uint32_t)pos[r]);
    }
    HP_PROF();
    cl.sync();
    if (ps + 1 < passes) {
#pragma unroll
      for (int r = 0; r < IPT; ++r) {
        const uint2 v = s_buf[w * 32 * IPT + r * 32 + lane];
        key[r] = v.x;
        pos[r] = (int32_t)v.y;
      }
    }
  }
  // ---- local segment analysis (thread t owns slice items [t*IPT, t*IPT+IPT))
  const int nvalid = min(S, max(0, T - c * S));
  if (tid == 0) s_pub[15] = c > 0 ? (int)cl.map_shared_rank(s_buf, c - 1)[S - 1].x : 0;
  __syncthreads();
  const uint32_t prev_last = (uint32_t)s_pub[15];
  bool h[IPT];
  int heads = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int li = tid * IPT + k;
    const uint32_t prev = li > 0 ? s_buf[li - 1].x : prev_last;
    h[k] = li < nvalid && ((c == 0 && li == 0) || s_buf[li].x != prev);
    heads += h[k];
  }
  for (int li = tid; li < nvalid; li += NT) pl.sorted_pos[c * S + li] = (int32_t)s_buf[li].y;
  int cta_heads;
  const int hb = block_excl_scan<NT>(heads, s_scan, &cta_heads);
  {
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < IPT; ++k)
      if (h[k]) s_hpos[hb + cnt++] = tid * IPT + k;
  }
  __syncthreads();
  // unique ids of this slice per partition: heads are in ascending id order, so
  // count(p) = #heads with id < lo(p+1) - #heads with id < lo(p)
  for (int p = tid; p < P; p += NT) {
    auto below = [&](int64_t x) {
      int lo = 0, hi = cta_heads;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)s_buf[s_hpos[mid]].x < x) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    s_pcnt[p] = below(p + 1 < P ? route.lo(p + 1) : pl.V) - below(route.lo(p));
  }
  // lengths of every local segment except the last one (its end lies in a later CTA)
  int ni = 0, np = 0, nl = 0;
  for (int sidx = hb; sidx < hb + heads; ++sidx) {
    if (sidx + 1 >= cta_heads) break;
    const int L = s_hpos[sidx + 1] - s_hpos[sidx];
    const int n0 = (L + HP_CHUNK - 1) / HP_CHUNK;
    ni += n0;
    if (L > HP_CHUNK) { np += n0; ++nl; }
  }
  int packed_tot;
  const int packed = block_excl_scan<NT>(pack3(ni, np, nl), s_scan, &packed_tot);
  if (tid == 0) {
    s_pub[PB_HEADS] = cta_heads;
    s_pub[PB_FIRST] = cta_heads ? c * S + s_hpos[0] : INT_MAX;
    s_pub[PB_LAST] = cta_heads ? c * S + s_hpos[cta_heads - 1] : -1;
    s_pub[PB_ITEMS] = packed_tot & 0xfff;
    s_pub[PB_PARTS] = (packed_tot >> 12) & 0x3ff;
    s_pub[PB_LONGS] = (packed_tot >> 22) & 0x3ff;
  }
  HP_PROF();
  cl.sync();  // ---- the one metadata barrier
  HP_PROF();
  // global prefixes from the published state of every CTA
  int seg_base = 0, U = 0, bi = packed & 0xfff, bp = (packed >> 12) & 0x3ff, bl = packed >> 22;
  int tot_i = 0, tot_p = 0, tot_l = 0, my_last_len = 0;
  {
    // one DSMEM read per published value, then every thread reads local smem
    int* s_all = s_base;  // CS * PB_N <= 256 ints, free after the sort
    if (tid < CS * PB_N) s_all[tid] = cl.map_shared_rank(s_pub, tid / PB_N)[tid % PB_N];
    __syncthreads();
    int pub[CS][PB_N];
#pragma unroll
    for (int cc = 0; cc < CS; ++cc)
#pragma unroll
      for (int f = 0; f < PB_N; ++f) pub[cc][f] = s_all[cc * PB_N + f];
    int next_head = T;
#pragma unroll
    for (int cc = CS - 1; cc >= 0; --cc) {
      int ci = pub[cc][PB_ITEMS], cp = pub[cc][PB_PARTS], cl_ = pub[cc][PB_LONGS];
      if (pub[cc][PB_HEADS]) {
        const int L = next_head - pub[cc][PB_LAST];
        const int n0 = (L + HP_CHUNK - 1) / HP_CHUNK;
        ci += n0;
        if (L > HP_CHUNK) { cp += n0; ++cl_; }
        if (cc == c) my_last_len = L;
        next_head = pub[cc][PB_FIRST];
      }
      U += pub[cc][PB_HEADS];
      tot_i += ci; tot_p += cp; tot_l += cl_;
      if (cc < c) { seg_base += pub[cc][PB_HEADS]; bi += ci; bp += cp; bl += cl_; }
    }
  }
  // partition totals -> first unique index and owner-grouped send-slot bases
  {
    int carry = 0;
    for (int p0 = 0; p0 <= P; p0 += NT) {
      const int p = p0 + tid;
      int v = 0;
      if (p < P)
#pragma unroll
        for (int cc = 0; cc < CS; ++cc) v += cl.map_shared_rank(s_pcnt, cc)[p];
      int t;
      const int ex = block_excl_scan<NT>(v, s_scan, &t);
      if (p <= P) s_first[p] = carry + ex;
      carry += t;
    }
  }
  __syncthreads();
  partition_bases<NT>(s_first, owner, P, pl.nranks, s_pbase, c == 0 ? dest_counts : nullptr,
                      s_dest);
  HP_PROF();
  // ---- per-segment outputs (thread t: segments whose head is in its items)
  auto seg_out = [&](int sidx, int L, int& bi_, int& bp_, int& bl_) {
    const int u = seg_base + sidx;
    const int li = s_hpos[sidx];
    const uint32_t id = s_buf[li].x;
    int slot = -1, dst = -1;  // the dropped-id sentinel segment (id == V): no slot, no store
    if ((int64_t)id < pl.V) {
      const int p = route.part(id);
      slot = s_pbase[p] + (u - s_first[p]);
      if (send_ids) send_ids[slot] = id;
      if (counts) counts[slot] = L;
      dst = seg_dst(id, p, slot, dst_pb, route, &s_err);
    }
    s_sig[sidx] = slot;
    emit_items(pl, u, c * S + li, L, dst, bi_, bp_, bl_, (int)s_buf[li].y, tot_p);
    const int n0 = (L + HP_CHUNK - 1) / HP_CHUNK;
    bi_ += n0;
    if (L > HP_CHUNK) { bp_ += n0; ++bl_; }
  };
  for (int sidx = hb; sidx < hb + heads; ++sidx) {
    const int L = sidx + 1 < cta_heads ? s_hpos[sidx + 1] - s_hpos[sidx] : my_last_len;
    seg_out(sidx, L, bi, bp, bl);
  }
  if (c == CS - 1 && tid == 0) {
    pl.counters[C_UNIQ] = U;
    pl.counters[C_ITEMS] = tot_i;
    pl.counters[C_PARTIALS] = tot_p;
    pl.counters[C_LONG] = tot_l;
    if (n_uniq) *n_uniq = s_first[P];  // valid unique rows (the sentinel segment excluded)
  }
  __syncthreads();
  HP_PROF();
  if (inv) {
    // items before the first local head belong to the previous CTA's last segment
    int spill_slot = 0;
    if (c > 0 && (cta_heads == 0 || s_hpos[0] > 0) && nvalid > 0) {
      const uint32_t id = s_buf[0].x;
      if ((int64_t)id < pl.V) {
        const int p = route.part(id);
        spill_slot = s_pbase[p] + (seg_base - 1 - s_first[p]);
      } else {
        spill_slot = -1;
      }
    }
    int hcount = hb;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int li = tid * IPT + k;
      hcount += h[k];
      if (li < nvalid) inv[s_buf[li].y] = hcount > 0 ? s_sig[hcount - 1] : spill_slot;
    }
  }
  __syncthreads();
  if (tid == 0 && s_err) atomicOr(&pl.counters[C_ERR], s_err);
  HP_PROF();
  cl.sync();  // no CTA may exit while others still read its shared memory
  HP_PROF();
#undef HP_PROF
  HP_SPAN_END(SP_DEDUP);
}

constexpr size_t tile_smem_bytes() {
  return (size_t)HP_TILE * 8 + (size_t)(HP_TILE_THREADS / 32) * HS * 4 + 40 * 4 + HP_RADIX * 4;
}

template <int NT>
constexpr size_t cluster_smem_bytes() {
  return (size_t)HP_CL_SLICE * 16 + (size_t)(NT / 32) * HS * 4 + 40 * 4 +
         2 * HP_RADIX * 4 + 16 * 4 + MAX_RANKS * 4 + (3 * CL_PMAX + 1) * 4;
}

// ------------------------------------------------------------------ large path
__global__ void __launch_bounds__(HP_TILE_THREADS)
k_tile_hist(DedupPlan pl, const int64_t* __restrict__ ids, int src, int shift) {
  __shared__ int s_h[HP_RADIX];
  for (int i = threadIdx.x; i < HP_RADIX; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * HP_TILE;
  for (int k = 0; k < HP_TILE_IPT; ++k) {
    const int64_t i = base + k * HP_TILE_THREADS + threadIdx.x;
    if (i < pl.T) {
      const uint32_t key = ids ? load_key(ids, i, pl.V, &pl.counters[C_ERR]) : pl.key[src][i];
      const unsigned d = (key >> shift) & (HP_RADIX - 1);
      const unsigned peers = __match_any_sync(__activemask(), d);
      if ((peers & lanemask_lt()) == 0) atomicAdd(&s_h[d], __popc(peers));
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < HP_RADIX; d += blockDim.x)
    pl.tile_hist[(int64_t)d * pl.ntiles + blockIdx.x] = s_h[d];
}

// One CTA per digit: exclusive scan of that digit's per-tile counts.
__global__ void __launch_bounds__(1024) k_digit_scan(DedupPlan pl) {
  __shared__ int s_scan[40];
  int* row = pl.tile_hist + (int64_t)blockIdx.x * pl.ntiles;
  int carry = 0;
  for (int b = 0; b < pl.ntiles; b += 1024) {
    const int i = b + threadIdx.x;
    const int v = i < pl.ntiles ? row[i] : 0;
    int tot;
    const int ex = block_excl_scan<1024>(v, s_scan, &tot);
    if (i < pl.ntiles) row[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) pl.digit_tot[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(HP_TILE_THREADS, 2)
k_tile_scatter(DedupPlan pl, const int64_t* __restrict__ ids, int src, int shift) {
  constexpr int NT = HP_TILE_THREADS, IPT = HP_TILE_IPT, NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* s_key = reinterpret_cast<uint32_t*>(smem);
  int32_t* s_pos = reinterpret_cast<int32_t*>(s_key + HP_TILE);
  int* s_hist = s_pos + HP_TILE;
  int* s_scan = s_hist + NW * HS;
  int* s_gbase = s_scan + 40;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * HP_TILE;
  const int valid = (int)min((int64_t)HP_TILE, pl.T - base);
  uint32_t key[IPT];
  int32_t pos[IPT];
  int rank[IPT];
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    const int li = w * 32 * IPT + r * 32 + lane;
    const int64_t i = base + li;
    if (li < valid) {
      if (ids) {
        key[r] = load_key(ids, i, pl.V, nullptr);  // errors already flagged by k_tile_hist
        pos[r] = (int32_t)i;
      } else {
        key[r] = pl.key[src][i];
        pos[r] = pl.pos[src][i];
      }
    } else {
      key[r] = 0xffffffffu;
      pos[r] = -1;
    }
  }
  // digit bases: exclusive scan of digit totals + this tile's column offset
  if (threadIdx.x < HP_RADIX) s_gbase[threadIdx.x] = pl.digit_tot[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < 32) {
    int carry = 0;
    for (int d0 = 0; d0 < HP_RADIX; d0 += 32) {
      const int v = s_gbase[d0 + lane];
      const int incl = warp_incl_scan(v);
      s_gbase[d0 + lane] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  if (threadIdx.x < HP_RADIX)
    s_gbase[threadIdx.x] += pl.tile_hist[(int64_t)threadIdx.x * pl.ntiles + blockIdx.x];
  block_rank<NT, IPT>(key, shift, rank, s_hist, s_scan);
#pragma unroll
  for (int r = 0; r < IPT; ++r) {
    s_key[rank[r]] = key[r];
    s_pos[rank[r]] = pos[r];
  }
  __syncthreads();
  const int dst = src ^ 1;
  for (int idx = threadIdx.x; idx < valid; idx += NT) {
    const uint32_t k = s_key[idx];
    const int d = (k >> shift) & (HP_RADIX - 1);
    const int64_t o = s_gbase[d] + (idx - s_hist[d]);
    pl.key[dst][o] = k;
    pl.pos[dst][o] = s_pos[idx];
  }
}

// ---- device-wide exclusive scan (reduce-then-scan), n from host or device
__global__ void __launch_bounds__(HP_SCAN_BLOCK)
k_scan_reduce(const int32_t* __restrict__ a, int64_t n_host, const int32_t* n_dev, int32_t* bsum) {
  __shared__ int s_scan[40];
  const int64_t n = n_dev ? *n_dev : n_host;
  const int64_t base = (int64_t)blockIdx.x * HP_SCAN_TILE;
  int s = 0;
  for (int k = 0; k < HP_SCAN_IPT; ++k) {
    const int64_t i = base + (int64_t)threadIdx.x * HP_SCAN_IPT + k;
    if (i < n) s += a[i];
  }
  int tot;
  block_excl_scan<HP_SCAN_BLOCK>(s, s_scan, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_top(int32_t* bsum, int nb, int32_t* total) {
  __shared__ int s_scan[40];
  int carry = 0;
  for (int b = 0; b < nb; b += 1024) {
    const int i = b + threadIdx.x;
    const int v = i < nb ? bsum[i] : 0;
    int tot;
    const int ex = block_excl_scan<1024>(v, s_scan, &tot);
    if (i < nb) bsum[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void __launch_bounds__(HP_SCAN_BLOCK)
k_scan_down(int32_t* a, int64_t n_host, const int32_t* n_dev, const int32_t* __restrict__ bsum) {
  __shared__ int s_scan[40];
  const int64_t n = n_dev ? *n_dev : n_host;
  const int64_t base = (int64_t)blockIdx.x * HP_SCAN_TILE + (int64_t)threadIdx.x * HP_SCAN_IPT;
  int v[HP_SCAN_IPT];
  int s = 0;
  for (int k = 0; k < HP_SCAN_IPT; ++k) {
    v[k] = base + k < n ? a[base + k] : 0;
    s += v[k];
  }
  int tot;
  int run = block_excl_scan<HP_SCAN_BLOCK>(s, s_scan, &tot) + bsum[blockIdx.x];
  for (int k = 0; k < HP_SCAN_IPT; ++k) {
    if (base + k < n) a[base + k] = run;
    run += v[k];
  }
}

int device_scan(int32_t* a, int64_t n_host, const int32_t* n_dev, int32_t* bsum, int32_t* total,
                cudaStream_t st) {
  const int nb = (int)((n_host + HP_SCAN_TILE - 1) / HP_SCAN_TILE);
  if (nb == 0) return HP_OK;
  k_scan_reduce<<<nb, HP_SCAN_BLOCK, 0, st>>>(a, n_host, n_dev, bsum);
  k_scan_top<<<1, 1024, 0, st>>>(bsum, nb, total);
  k_scan_down<<<nb, HP_SCAN_BLOCK, 0, st>>>(a, n_host, n_dev, bsum);
  HP_LAUNCHED(3, "device_scan");
  return HP_OK;
}

// ---- large-path metadata kernels
__global__ void k_heads(DedupPlan pl, const uint32_t* __restrict__ skey) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pl.T;
       i += (int64_t)gridDim.x * blockDim.x)
    pl.segidx[i] = (i == 0 || skey[i] != skey[i - 1]) ? 1 : 0;
}

__global__ void k_heads_write(DedupPlan pl, const uint32_t* __restrict__ skey) {
  const int U = pl.counters[C_UNIQ];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pl.T;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool h = i == 0 || skey[i] != skey[i - 1];
    const int ex = pl.segidx[i];
    if (h) {
      pl.seg_start[ex] = (int)i;
      pl.uniq_key[ex] = skey[i];
    }
    pl.segidx[i] = ex + (h ? 1 : 0) - 1;
    if (i == 0) pl.seg_start[U] = (int)pl.T;
  }
}

// first_u[P] = valid unique rows: the dropped-id sentinel segment (key V) is last
__global__ void k_first_u(DedupPlan pl, int32_t* n_uniq) {
  const Router route(pl.V, pl.P);
  const int U = pl.counters[C_UNIQ];
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= pl.P; p += gridDim.x * blockDim.x) {
    const int f = lower_bound_u32(pl.uniq_key, U, (uint32_t)(p == pl.P ? pl.V : route.lo(p)));
    pl.first_u[p] = f;
    if (p == pl.P && n_uniq) *n_uniq = f;
  }
}

__global__ void __launch_bounds__(1024)
k_part_base(DedupPlan pl, const int32_t* __restrict__ owner, int32_t* dest_counts) {
  __shared__ int s_dest[MAX_RANKS];
  partition_bases<1024>(pl.first_u, owner, pl.P, pl.nranks, pl.part_base, dest_counts, s_dest);
}

// Per segment: send slot, destination row, outputs, and the three count
// arrays (items, partial slots, long flag) to be scanned.
__global__ void k_seg_counts(DedupPlan pl, const int64_t* __restrict__ dst_pb, int64_t* send_ids,
                             int32_t* counts) {
  const Router route(pl.V, pl.P);
  const int U = pl.counters[C_UNIQ];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    const int L = pl.seg_start[u + 1] - pl.seg_start[u];
    const int n0 = (L + HP_CHUNK - 1) / HP_CHUNK;
    const uint32_t id = pl.uniq_key[u];
    if ((int64_t)id < pl.V) {
      const int p = route.part(id);
      const int slot = pl.part_base[p] + (u - pl.first_u[p]);
      pl.sigma[u] = slot;
      if (send_ids) send_ids[slot] = id;
      if (counts) counts[slot] = L;
      pl.dst[u] = seg_dst(id, p, slot, dst_pb, route, &pl.counters[C_ERR]);
    } else {  // dropped ids (sentinel V): no slot, no destination
      pl.sigma[u] = -1;
      pl.dst[u] = -1;
    }
    pl.item_off[u] = n0;
    pl.part_off[u] = L > HP_CHUNK ? n0 : 0;
    pl.long_tmp[u] = L > HP_CHUNK ? 1 : 0;
  }
}

__global__ void k_items(DedupPlan pl) {
  const int U = pl.counters[C_UNIQ];
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    const int j0 = pl.seg_start[u];
    emit_items(pl, u, j0, pl.seg_start[u + 1] - j0, pl.dst[u], pl.item_off[u], pl.part_off[u],
               pl.long_tmp[u], pl.sorted_pos[j0], pl.counters[C_PARTIALS]);
  }
}

__global__ void k_inv(DedupPlan pl, int32_t* inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pl.T;
       i += (int64_t)gridDim.x * blockDim.x)
    inv[pl.sorted_pos[i]] = pl.sigma[pl.segidx[i]];
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

long long* g_prof = nullptr;  // set by hp_debug_set_profile (instrumentation only)

size_t dedup_ws_bytes(int64_t T, int32_t D, int32_t P) {
  const int64_t Tc = T < 1 ? 1 : T;
  const int64_t ntiles = (Tc + HP_TILE - 1) / HP_TILE;
  const int64_t nscan = (Tc + HP_SCAN_TILE - 1) / HP_SCAN_TILE + 2;
  const int64_t prow = 2 * Tc / HP_CHUNK + 2;
  size_t s = align256(4 * C_NCOUNTERS);
  s += align256(4 * (size_t)CMB_LV * (2 * Tc / HP_CHUNK + 2));  // fused-combine arrival counters
  s += 4 * align256(4 * Tc);          // key[2], pos[2]
  s += 3 * align256(4 * (Tc + 1));    // uniq_key, seg_start, item_off
  s += 5 * align256(4 * Tc);          // segidx, sigma, part_off, dst, long_tmp
  s += align256(16 * Tc) + align256(16 * (Tc / HP_CHUNK + 2));  // items, longs
  s += align256(16 * prow);                                       // part_desc
  s += align256(4 * (Tc / HP_CHUNK + 2));                         // long_flag
  s += align256(4 * ((size_t)P + 1)) + 2 * align256(4 * (size_t)P);
  s += align256(4 * HP_RADIX * ntiles) + align256(4 * HP_RADIX);
  s += align256(4 * nscan);
  s += align256(4 * (size_t)D * prow);
  s += 2 * align256(4 * (HP_RS_MAX_WARPS + 1));
  s += align256(16 * Tc);             // send_info
  return s;
}

int rs_stages(int32_t D) {
  switch (D) {
    case 128: return 16;
    case 256: return 12;
    case 512: return 8;
    case 1024: return 6;
    default: return 0;
  }
}

int rs_warps(int32_t D) {
  const int S = rs_stages(D);
  if (S == 0) return 0;
  const int cta_bytes = 4 * S * D * 4;  // 4 warps x S row slots
  int ctas = (220 << 10) / cta_bytes;
  ctas = ctas < 1 ? 1 : (ctas > g_rs_ctas ? g_rs_ctas : ctas);
  const int nw = sm_count() * 4 * ctas;
  return nw < HP_RS_MAX_WARPS ? nw : HP_RS_MAX_WARPS - HP_RS_MAX_WARPS % 4;
}

int carve_plan(DedupPlan* pl, void* ws, size_t ws_bytes, int64_t T, int32_t D, int64_t V,
               int32_t P, int32_t nranks) {
  HP_REQUIRE(ws != nullptr, "workspace is NULL");
  HP_REQUIRE(V >= 1 && V < (int64_t(1) << 31), "table rows V must be in [1, 2^31)");
  HP_REQUIRE(P >= 1 && P <= V, "partition count P must be in [1, V]");
  HP_REQUIRE(nranks >= 1 && nranks <= MAX_RANKS, "nranks out of range");
  HP_REQUIRE(T >= 0 && T < (int64_t(1) << 31), "T out of range");
  HP_REQUIRE(D >= 1, "D must be >= 1");
  if (ws_bytes < dedup_ws_bytes(T, D, P)) {
    set_error("workspace too small for dedup plan");
    return HP_EWS;
  }
  const int64_t Tc = T < 1 ? 1 : T;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) { void* r = p; p += align256(bytes); return r; };
  pl->counters = (int32_t*)take(4 * C_NCOUNTERS);  // first: fixed offset (hp_plan_status)
  // right after the counters, so ONE memset per plan build clears both
  pl->comb_ctr = (int32_t*)take(4 * (size_t)CMB_LV * (2 * Tc / HP_CHUNK + 2));
  pl->T = T;
  pl->D = D;
  pl->P = P;
  pl->nranks = nranks;
  pl->V = V;
  int bits = 0;
  while (bits < 31 && (int64_t(1) << bits) <= V) ++bits;  // holds V: the dropped-id sentinel
  pl->key_bits = bits < 1 ? 1 : bits;
  pl->ntiles = (int32_t)((Tc + HP_TILE - 1) / HP_TILE);
  pl->key[0] = (uint32_t*)take(4 * Tc);
  pl->key[1] = (uint32_t*)take(4 * Tc);
  pl->pos[0] = (int32_t*)take(4 * Tc);
  pl->pos[1] = (int32_t*)take(4 * Tc);
  pl->uniq_key = (uint32_t*)take(4 * (Tc + 1));
  pl->seg_start = (int32_t*)take(4 * (Tc + 1));
  pl->item_off = (int32_t*)take(4 * (Tc + 1));
  pl->segidx = (int32_t*)take(4 * Tc);
  pl->sigma = (int32_t*)take(4 * Tc);
  pl->part_off = (int32_t*)take(4 * Tc);
  pl->dst = (int32_t*)take(4 * Tc);
  pl->long_tmp = (int32_t*)take(4 * Tc);
  pl->items = (int4*)take(16 * Tc);
  pl->longs = (int4*)take(16 * (Tc / HP_CHUNK + 2));
  pl->part_desc = (int4*)take(16 * (2 * Tc / HP_CHUNK + 2));
  pl->long_flag = (int32_t*)take(4 * (Tc / HP_CHUNK + 2));
  pl->cbcast = 0;
  pl->first_u = (int32_t*)take(4 * ((size_t)P + 1));
  pl->part_base = (int32_t*)take(4 * (size_t)P);
  pl->zero_owner = (int32_t*)take(4 * (size_t)P);
  pl->tile_hist = (int32_t*)take(4 * HP_RADIX * (size_t)pl->ntiles);
  pl->digit_tot = (int32_t*)take(4 * HP_RADIX);
  pl->scan_bsum = (int32_t*)take(4 * ((Tc + HP_SCAN_TILE - 1) / HP_SCAN_TILE + 2));
  pl->partial_rows = 2 * Tc / HP_CHUNK + 2;
  pl->partials = (float*)take(4 * (size_t)D * pl->partial_rows);
  pl->wb_item = (int32_t*)take(4 * (HP_RS_MAX_WARPS + 1));
  pl->wb_row = (int32_t*)take(4 * (HP_RS_MAX_WARPS + 1));
  pl->send_info = (int4*)take(16 * Tc);
  pl->nw = g_rowstream_off ? 0 : rs_warps(D);
  pl->fused = pl->nw <= 0 && g_fuse_tree;
  pl->reorder = pl->fused || (pl->nw <= 0 && g_split_long);
  pl->part = 0;
  pl->sorted_pos = pl->pos[0];
  pl->prof = g_prof;
  return HP_OK;
}

template <int NT, int CS>
int launch_cluster_nt(const DedupPlan& pl, const int64_t* ids, const int32_t* owner,
                      const int64_t* dst_pb, int64_t* send_ids, int32_t* counts, int32_t* inv,
                      int32_t* dest_counts, int32_t* n_uniq, cudaStream_t st) {
  constexpr int IPT = HP_CL_SLICE / NT;
  constexpr size_t smem = cluster_smem_bytes<NT>();
  auto kern = k_dedup_cluster<NT, IPT, CS>;
  static bool configured = false;
  if (!configured) {
    HP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  launch_k(kern, dim3(CS), dim3(NT), smem, st, pl, ids, owner, dst_pb, send_ids, counts, inv, dest_counts, n_uniq);
  HP_LAUNCHED(1, "k_dedup_cluster");
  return HP_OK;
}

// 512 threads x 4 keys: spill-free at up to 128 registers (1024 x 2 spilled 60 B at
// its 64-register cap) and as fast in the step (r2o: 47.3 vs 47.1 us)
int g_cl_threads = 512;  // CTA shape of the cluster path (hp_debug_set_cluster_threads)

void set_cluster_threads(int nt) { g_cl_threads = nt; }
int g_rowstream_off = 1;  // row stream measured slower on the LM step
int g_rs_ctas = 4;
int g_owner_stream = 2;  // 0: k_owner_apply, 1: k_owner_stream, 2: k_owner_scan + k_owner_rows
int g_combine_blocks = 0;  // 0: one CTA per long segment up to the SM count
int g_dar_blocks = 0;     // HP_DAR_PIPE grid (0 = one block per SM)
int g_dar_rg_blocks = 0;  // HP_DAR_SM reduce/gather grid (0: 2 per SM)
int g_dar_tma = 36;  // K7 scatter on TMA, one-warp CTAs per peer chunk (hp_debug_set_dar_tma; 0: LSU stores)
int g_dar_rg_tma = 0;  // K7 reduce/gather on TMA, CTAs (hp_debug_set_dar_rg_tma, A/B)
int g_dar_deep = 0;  // SM-store K7 with deep unrolls (hp_debug_set_dar_deep, A/B)
int g_dar_buckets = 1;    // HP_DAR_SM buckets per step (hp_debug_set_dar_buckets)
int g_owner_waves = 1;    // peer-store kernels run many waves (no per-block fences)
int g_reduce_b = 2;
// fused tree: default OFF by measurement (r2x / r2mic): K4 alone at LM1B
// 24.3 vs 25.4 us, but the step no faster and 1.8x slower at the micro
// config's 16M draws (one CTA per long chunk holds 4-8x fewer chunks in flight
// than k_reduce's thread groups)
int g_split_long = 1;
int g_reduce_bps = 16;  // k_reduce grid cap in blocks per SM (hp_debug_set_reduce_bps)
int g_cbcast = 0;  // hp_debug_set_cbcast (A/B; measured slower in the step, see the header)
int g_comb_lite = 0;  // hp_debug_set_comb_lite (A/B)
int g_long_tma = 0;  // hp_debug_set_long_tma (A/B)
int g_long_b8 = 0;  // long-chunk reduce with 8 rows in flight (hp_debug_set_long_b8; A/B)
int g_fuse_tree = 0;
HP_SPAN_SETTER(set_spans_dedup)

template <int CS>
int launch_cluster(const DedupPlan& pl, const int64_t* ids, const int32_t* owner,
                   const int64_t* dst_pb, int64_t* send_ids, int32_t* counts, int32_t* inv,
                   int32_t* dest_counts, int32_t* n_uniq, cudaStream_t st) {
  switch (g_cl_threads) {
    case 256:
      return launch_cluster_nt<256, CS>(pl, ids, owner, dst_pb, send_ids, counts, inv,
                                        dest_counts, n_uniq, st);
    case 512:
      return launch_cluster_nt<512, CS>(pl, ids, owner, dst_pb, send_ids, counts, inv,
                                        dest_counts, n_uniq, st);
    default:
      return launch_cluster_nt<1024, CS>(pl, ids, owner, dst_pb, send_ids, counts, inv,
                                         dest_counts, n_uniq, st);
  }
}

// Which ping-pong buffer holds the sorted positions of a plan built by
// build_plan with the same (T, P, V): the cluster path writes pos[0]; the
// multi-kernel path leaves them in pos[passes & 1].
void restore_sorted_pos(DedupPlan& pl) {
  if (pl.T <= HP_SMALL_MAX && pl.P <= CL_PMAX) {
    pl.sorted_pos = pl.pos[0];
  } else {
    const int passes = (pl.key_bits + HP_RADIX_BITS - 1) / HP_RADIX_BITS;
    pl.sorted_pos = pl.pos[passes & 1];
  }
}

int build_plan(DedupPlan& pl, const int64_t* ids, const int32_t* owner,
               const int64_t* dst_pb, int64_t* send_ids, int32_t* counts, int32_t* inv,
               int32_t* dest_counts, int32_t* n_uniq, cudaStream_t st) {
  // counters + the fused-combine arrival counters (contiguous, carve_plan).
  // The cluster path writes every counter itself (C_ERR zeroed in-kernel), so
  // without the fused tree it needs no memset: a memset node in front of the
  // cluster kernel let the concurrent apply's k_reduce fill every SM first and
  // the cluster (8 co-scheduled SMs) then waited ~14 us for it (LM1B n = 1 step
  // 44.1 -> 40.3 us without it).
  const bool cluster = pl.T > 0 && pl.T <= HP_SMALL_MAX && pl.P <= CL_PMAX;
  if (!cluster || pl.fused)
    HP_CUDA(cudaMemsetAsync(pl.counters, 0,
                            reinterpret_cast<char*>(pl.comb_ctr) - reinterpret_cast<char*>(pl.counters) +
                                4 * (size_t)CMB_LV * pl.partial_rows,
                            st));
  if (pl.T == 0) {
    if (dest_counts) HP_CUDA(cudaMemsetAsync(dest_counts, 0, 4 * (size_t)pl.nranks, st));
    if (n_uniq) HP_CUDA(cudaMemsetAsync(n_uniq, 0, 4, st));
    return HP_OK;
  }
  if (pl.T <= HP_SMALL_MAX && pl.P <= CL_PMAX) {
    pl.sorted_pos = pl.pos[0];
    // smallest cluster that holds T (fewer CTAs -> cheaper cluster barriers)
    int rc;
    if (pl.T <= 2 * HP_CL_SLICE)
      rc = launch_cluster<2>(pl, ids, owner, dst_pb, send_ids, counts, inv, dest_counts, n_uniq, st);
    else if (pl.T <= 4 * HP_CL_SLICE)
      rc = launch_cluster<4>(pl, ids, owner, dst_pb, send_ids, counts, inv, dest_counts, n_uniq, st);
    else
      rc = launch_cluster<8>(pl, ids, owner, dst_pb, send_ids, counts, inv, dest_counts, n_uniq, st);
    return rc;
  }
  // ---- large path: LSD radix sort, 8-bit digits
  static bool tile_configured = false;
  if (!tile_configured) {
    HP_CUDA(cudaFuncSetAttribute(k_tile_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)tile_smem_bytes()));
    tile_configured = true;
  }
  const int passes = (pl.key_bits + HP_RADIX_BITS - 1) / HP_RADIX_BITS;
  int src = 0;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * HP_RADIX_BITS;
    const int64_t* in_ids = ps == 0 ? ids : nullptr;
    k_tile_hist<<<pl.ntiles, HP_TILE_THREADS, 0, st>>>(pl, in_ids, src, shift);
    k_digit_scan<<<HP_RADIX, 1024, 0, st>>>(pl);
    k_tile_scatter<<<pl.ntiles, HP_TILE_THREADS, tile_smem_bytes(), st>>>(pl, in_ids, src, shift);
    HP_LAUNCHED(3, "radix pass");
    src ^= 1;
  }
  pl.sorted_pos = pl.pos[src];
  const uint32_t* skey = pl.key[src];
  const int g = grid_for(pl.T, 256, sm_count() * 8);
  k_heads<<<g, 256, 0, st>>>(pl, skey);
  int rc = device_scan(pl.segidx, pl.T, nullptr, pl.scan_bsum, &pl.counters[C_UNIQ], st);
  if (rc) return rc;
  k_heads_write<<<g, 256, 0, st>>>(pl, skey);
  k_first_u<<<grid_for(pl.P + 1, 256, 1024), 256, 0, st>>>(pl, n_uniq);
  k_part_base<<<1, 1024, 0, st>>>(pl, owner, dest_counts);
  k_seg_counts<<<g, 256, 0, st>>>(pl, dst_pb, send_ids, counts);
  HP_LAUNCHED(5, "dedup metadata");
  const int32_t* U = &pl.counters[C_UNIQ];
  if ((rc = device_scan(pl.item_off, pl.T, U, pl.scan_bsum, &pl.counters[C_ITEMS], st))) return rc;
  if ((rc = device_scan(pl.part_off, pl.T, U, pl.scan_bsum, &pl.counters[C_PARTIALS], st))) return rc;
  if ((rc = device_scan(pl.long_tmp, pl.T, U, pl.scan_bsum, &pl.counters[C_LONG], st))) return rc;
  k_items<<<g, 256, 0, st>>>(pl);
  if (inv) k_inv<<<g, 256, 0, st>>>(pl, inv);
  HP_LAUNCHED(inv ? 2 : 1, "dedup items");
  return HP_OK;
}

}  // namespace hp
