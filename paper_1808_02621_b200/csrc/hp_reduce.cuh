// Segmented row reduction kernels shared by the local (reduce.cu) and the
// peer-memory (p2p.cu) paths; see reduce.cu for the summation tree.
#pragma once

#include <cooperative_groups.h>

#include "hp_dedup.cuh"

namespace hp {

// Epilogue contract:
//   Pre load(dst, c4)            issued before the row loads (depends on the item only)
//   void store(dst, c4, g, pre)  consumes the summed float4
//   kRemote                      stores go to peer memory: the caller launches
//                                k_publish (one block: system fence, then
//                                grid_done()) after k_combine; stream order makes
//                                every block's stores happen-before that fence, so
//                                the reduce / combine blocks do not fence or drain

// Epilogue interface: Pre load(dst, c4) is issued BEFORE the row loads (it
// only depends on the item), store(dst, c4, g, pre) consumes the summed float4.
struct EpiSend {
  static constexpr bool kRemote = false;
  static constexpr bool kOut = false;  // fused pull: the new row also goes to the positions
  static constexpr int kPre = 0;  // table rows the epilogue reads (row stream stages them)
  __device__ __forceinline__ const float4* pre_row(int, int) const { return nullptr; }
  float4* rows;
  int D4;
  struct Pre {};
  __device__ __forceinline__ Pre load(int, int) const { return {}; }
  __device__ __forceinline__ void store(int dst, int c4, float4 g, Pre) const {
    rows[(int64_t)dst * D4 + c4] = g;
  }
};

// Optimizer state a row update needs (only what the optimizer uses, so the
// prefetched epilogue operands stay in as few registers as possible).
template <int OPT> struct ApplyPre { float4 w, a, b; };
template <> struct ApplyPre<HP_OPT_SGD> { float4 w; };
template <> struct ApplyPre<HP_OPT_ADAGRAD> { float4 w, a; };

// field k of a Pre (0 = w, 1 = s0, 2 = s1)
template <class Pre>
__device__ __forceinline__ void set_pre(Pre& p, int k, float4 v) {
  if constexpr (sizeof(Pre) >= 16) { if (k == 0) p.w = v; }
  if constexpr (sizeof(Pre) >= 32) { if (k == 1) p.a = v; }
  if constexpr (sizeof(Pre) >= 48) { if (k == 2) p.b = v; }
}

template <int OPT>
struct EpiApply {
  static constexpr bool kRemote = false;
  static constexpr bool kOut = true;
  static constexpr int kPre = OPT == HP_OPT_SGD ? 1 : (OPT == HP_OPT_ADAGRAD ? 2 : 3);
  float4* w;
  float4* s0;
  float4* s1;
  hp_optim o;
  int D4;
  float4* out;  // fused pull (n = 1 steps): out[t] = new row, for every position t; or nullptr
  using Pre = ApplyPre<OPT>;

  __device__ __forceinline__ const float4* pre_row(int k, int dst) const {
    const float4* b = k == 0 ? w : (k == 1 ? s0 : s1);
    return b + (int64_t)dst * D4;
  }

  __device__ __forceinline__ Pre load(int dst, int c4) const {
    Pre p;
    const int64_t off = (int64_t)dst * D4 + c4;
    p.w = w[off];
    if constexpr (OPT != HP_OPT_SGD) p.a = s0[off];
    if constexpr (OPT == HP_OPT_ADAM) p.b = s1[off];
    return p;
  }

  __device__ __forceinline__ void upd(float& wv, float& a, float& b, float g) const {
    g = __fmul_rn(g, o.agg_scale);
    if (OPT == HP_OPT_SGD) {
      wv = __fsub_rn(wv, __fmul_rn(o.lr, g));
    } else if (OPT == HP_OPT_ADAGRAD) {
      a = __fadd_rn(a, __fmul_rn(g, g));
      wv = __fsub_rn(wv, __fdiv_rn(__fmul_rn(o.lr, g), __fsqrt_rn(a)));
    } else {
      a = __fadd_rn(__fmul_rn(o.beta1, a), __fmul_rn(o.one_minus_beta1, g));
      b = __fadd_rn(__fmul_rn(o.beta2, b), __fmul_rn(o.one_minus_beta2, __fmul_rn(g, g)));
      wv = __fsub_rn(wv, __fdiv_rn(__fmul_rn(adam_lr_t(o), a), __fadd_rn(__fsqrt_rn(b), o.eps)));
    }
  }

  // returns the new table row (for the fused pull)
  __device__ __forceinline__ float4 store(int dst, int c4, float4 g, Pre p) const {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if constexpr (OPT != HP_OPT_SGD) a = p.a;
    if constexpr (OPT == HP_OPT_ADAM) b = p.b;
    upd(p.w.x, a.x, b.x, g.x);
    upd(p.w.y, a.y, b.y, g.y);
    upd(p.w.z, a.z, b.z, g.z);
    upd(p.w.w, a.w, b.w, g.w);
    const int64_t off = (int64_t)dst * D4 + c4;
    w[off] = p.w;
    if constexpr (OPT != HP_OPT_SGD) s0[off] = a;
    if constexpr (OPT == HP_OPT_ADAM) s1[off] = b;
    return p.w;
  }
};

// Fused pull of a short item (n <= 16 rows of one id): the new row (or zeros
// for a dropped id) goes to each of the item's positions; lane j of each warp
// of the group holds position j (myp).
template <class Epi>
__device__ __forceinline__ void pull_store(const Epi& epi, int n, int myp, int c4, float4 v,
                                           int D4) {
  if constexpr (Epi::kOut) {
    if (epi.out == nullptr) return;
    for (int j = 0; j < n; ++j) {
      const int64_t p = __shfl_sync(0xffffffffu, myp, j);
      if (c4 < D4) epi.out[p * D4 + c4] = v;
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Staging buffer of the long chunks (TMA): static, 16 KB, shared with the
// short items' epilogue prefetch (s_pre), so k_reduce's shared memory per CTA
// does not grow (the next step's cluster dedup runs beside it on the same SMs).
constexpr int STAGE_F4 = 1024;
// Rows staged per TMA batch: 8 rows of 2 KB at D = 512 (a chunk = 2 batches).
__host__ __device__ constexpr int stage_rows(int D) {
  return STAGE_F4 * 4 / D >= HP_CHUNK ? HP_CHUNK : (STAGE_F4 * 4 / D > 0 ? STAGE_F4 * 4 / D : 1);
}

// One node of a long segment's summation tree, whole CTA: rows src[0..n) (row
// pointers from `row_of(j)`) are TMA-copied into s_stage (batches of SR rows,
// one elected lane per row), then every column is summed in row order from
// +0.0 and handed to `out(c4, acc)`. Callers __syncthreads() before reusing
// s_stage. Returns the next mbarrier parity.
template <int CPT, class RowOf, class Out>
__device__ __forceinline__ uint32_t cta_stage_sum(float4* s_stage, uint64_t* bar, uint32_t parity,
                                                  int n, int D4, int SR, RowOf row_of, Out out,
                                                  bool proxy_fence) {
  const int tid = threadIdx.x;
  const uint32_t rowbytes = (uint32_t)D4 * 16u;
  // (SR == HP_CHUNK for D <= 1024: one batch; wider rows take several)
  float4 acc[CPT];  // CPT = columns per thread (D4 <= 256 * CPT)
#pragma unroll
  for (int k = 0; k < CPT; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j0 = 0; j0 < n; j0 += SR) {
    const int nb = min(SR, n - j0);
    if (tid < 32) {
      if (proxy_fence) fence_proxy_async_global();
      if (tid == 0) mbar_expect_tx(bar, rowbytes * (uint32_t)nb);
      __syncwarp();
      for (int j = tid; j < nb; j += 32) bulk_g2s(s_stage + (size_t)j * D4, row_of(j0 + j), rowbytes, bar);
    }
    mbar_wait(bar, parity);
    parity ^= 1u;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int c4 = tid + k * 256;
      if (c4 < D4)
        for (int j = 0; j < nb; ++j) acc[k] = f4_add(acc[k], s_stage[(size_t)j * D4 + c4]);
    }
    if (j0 + nb < n) __syncthreads();  // the batch is consumed before the next lands
  }
#pragma unroll
  for (int k = 0; k < CPT; ++k)
    if (tid + k * 256 < D4) out(k, tid + k * 256, acc[k]);
  return parity;
}

// A long segment's chunk, the whole CTA (level 0 + the fused upper levels).
// The chunk's n <= 16 gradient rows are TMA-copied into shared memory in one
// batch and summed per column in row order (one DRAM round trip instead of
// n/B); the partial row goes to its slot. The CTA then arrives at its tree node:
// level-l node g sums level-(l-1) items [16g, 16g+16) in order; level-l item g
// lives in the slot of its first child (partial slot bp + g*16^l, rewritten
// only after every child was read, by the node's last arriver), so no extra
// storage. Each node's arrival counter is one atomic (stores; __syncthreads;
// fence + atomic by thread 0; last arriver: fence, then TMA reads of the
// children from L2). The node whose level holds <= 16 items is the root: its
// last arriver applies the epilogue (optimizer update / push). Same tree as
// oracle.tree_sum (sequential groups of 16 from +0.0, then again on the group
// sums) and as k_combine. Long chunks are the first items (dedup.cu
// emit_items), so the hot ids' trees close in k_reduce's first wave.
template <int CPT, class Epi>
__device__ __forceinline__ uint32_t long_chunk(const DedupPlan& pl, const float4* vals, const Epi& epi,
                                               int lit, float4* s_stage, uint64_t* bar,
                                               uint32_t parity, int* s_bc) {
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  const int D4 = pl.D >> 2;
  const int SR = stage_rows(pl.D);
  const int tid = threadIdx.x;
  const int4 item = pl.items[lit];
  const int j0 = item.x, slot = item.z;
  const int4 d = pl.longs[-item.w - 1];  // {bp, n0, dst, u}
  const int64_t bp = d.x;
  parity = cta_stage_sum<CPT>(
      s_stage, bar, parity, item.y, D4, SR,
      [&](int j) { return vals + (int64_t)pl.sorted_pos[j0 + j] * D4; },
      [&](int, int c4, float4 a) { partials[(int64_t)slot * D4 + c4] = a; }, false);
  int i = slot - d.x, n_prev = d.y, lev = 1;
#pragma unroll 1
  while (true) {
    const bool root = n_prev <= HP_CHUNK;
    const int g = root ? 0 : i / HP_CHUNK;
    const int first = g * HP_CHUNK, nch = min(HP_CHUNK, n_prev - first);
    const int64_t node = bp + ((int64_t)g << (4 * lev));  // this node's item slot
    int* ctr = pl.comb_ctr + node * CMB_LV + (lev - 1);
    __syncthreads();  // every partial store of the CTA issued; s_stage consumed
    if (tid == 0) {
      __threadfence();
      s_bc[0] = atomicAdd(ctr, 1) == nch - 1;
    }
    __syncthreads();
    if (!s_bc[0]) break;
    __threadfence();
    const int64_t cs = (int64_t)1 << (4 * (lev - 1));  // child stride in slots
    typename Epi::Pre pre[CPT];
    if (root && d.z >= 0) {
#pragma unroll
      for (int k = 0; k < CPT; ++k)
        if (tid + k * 256 < D4) pre[k] = epi.load(d.z, tid + k * 256);
    }
    parity = cta_stage_sum<CPT>(
        s_stage, bar, parity, nch, D4, SR,
        [&](int j) { return partials + (bp + (int64_t)(first + j) * cs) * D4; },
        [&](int k, int c4, float4 a) {
          if (!root)
            partials[node * D4 + c4] = a;
          else if (d.z >= 0)
            epi.store(d.z, c4, a, pre[k]);
        },
        true);
    if (tid == 0) *ctr = 0;  // every arrival is in: reset for the plan's next apply
    if (root) break;
    i = g;
    n_prev = (n_prev + HP_CHUNK - 1) / HP_CHUNK;
    ++lev;
  }
  __syncthreads();  // s_stage / s_bc free for the next chunk
  return parity;
}

// Level 0 of the summation tree. A group of TPI threads owns an item
// {j0, n <= HP_CHUNK, dst, final}; each thread owns VPT float4 columns
// (c4 = lane-in-group + k*TPI). Row positions are loaded once per warp and
// broadcast by shuffle; B rows x VPT columns are in flight per thread before
// the in-order fp32 adds. Final items run the epilogue (its table-row loads
// are issued together with the positions); long-segment chunks write a
// partial row for k_combine. Small groups + <= 64 registers keep many items
// in flight per SM: the kernel is latency-bound on the item chain
// (descriptor -> positions/table rows -> gradient rows).
template <int TPI, int VPT, class Epi>
__host__ __device__ constexpr bool reduce_smem_pre() {
  return Epi::kPre > 0 && VPT <= 2 && (256 / TPI) * Epi::kPre * TPI * VPT * 16 <= 32768;
}

template <int TPI, int VPT, int B, class Epi>
__global__ void __launch_bounds__(256, reduce_smem_pre<TPI, VPT, Epi>() && Epi::kPre < 3 ? 4 : 3)
k_reduce(DedupPlan pl, const float* __restrict__ vals_f, Epi epi) {
  const float4* __restrict__ vals = reinterpret_cast<const float4*>(vals_f);
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  const int D4 = pl.D >> 2;
  constexpr int GPB = 256 / TPI;
  const int q = threadIdx.x % TPI;
  const int lane = threadIdx.x & 31;
  const int span_id = pl.part == 2 ? SP_REDUCE2 : SP_REDUCE;
  HP_ENTRY(span_id);
  // The epilogue's table rows (w, optimizer state) are staged through shared
  // memory with cp.async (each thread copies and later reads only its own
  // columns) instead of registers: ~16 fewer registers per thread at LM shapes.
  constexpr int KP = Epi::kPre;
  constexpr bool SP = reduce_smem_pre<TPI, VPT, Epi>();
  constexpr int NPRE = SP ? GPB * KP * VPT * TPI : 1;
  // long chunks: [stage_rows][D4] TMA staging; then the short items' s_pre
  __shared__ __align__(128) float4 s_buf[NPRE > STAGE_F4 ? NPRE : STAGE_F4];
  float4* s_pre = s_buf;
  float4* s_stage = s_buf;
  __shared__ uint64_t s_bar;
  __shared__ int s_bc[1];
  float4* my_pre = s_pre + (threadIdx.x / TPI) * KP * VPT * TPI + q;  // [g][k][v][TPI]
  const int n_items = pl.counters[C_ITEMS];
  auto process = [&](int it) -> int4 {
    const int4 item = pl.items[it];
    const int j0 = item.x, n = item.y, dst = item.z;
    const bool fin = item.w > 0;  // < 0: chunk of long segment -w-1 (fused combine)
    typename Epi::Pre pre[SP ? 1 : VPT];
    if (fin && dst >= 0) {
      if constexpr (SP) {
#pragma unroll
        for (int k = 0; k < KP; ++k)
#pragma unroll
          for (int v = 0; v < VPT; ++v)
            if (q + v * TPI < D4)
              cp_async16(my_pre + (k * VPT + v) * TPI, epi.pre_row(k, dst) + q + v * TPI);
        cp_async_commit();
      } else {
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (q + v * TPI < D4) pre[v] = epi.load(dst, q + v * TPI);
      }
    }
    // single-row items carry the row's position directly (item.x = -(pos+1))
    const int myp = j0 < 0 ? -j0 - 1 : (lane < n ? pl.sorted_pos[j0 + lane] : 0);
    float4 acc[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int jb = 0; jb < n; jb += B) {
      float4 x[B][VPT];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        const int64_t rb = (int64_t)__shfl_sync(0xffffffffu, myp, jb + e) * D4;
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (jb + e < n && q + v * TPI < D4) x[e][v] = ldg_stream(vals + rb + q + v * TPI);
      }
#pragma unroll
      for (int e = 0; e < B; ++e)
#pragma unroll
        for (int v = 0; v < VPT; ++v)
          if (jb + e < n) acc[v] = f4_add(acc[v], x[e][v]);
    }
    if constexpr (SP) {
      if (fin && dst >= 0) cp_async_wait<0>();
    }
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c4 = q + v * TPI;
      float4 nw = make_float4(0.f, 0.f, 0.f, 0.f);  // the pulled row (zeros: dropped id)
      if (c4 < D4) {
        if (fin) {
          if (dst >= 0) {
            typename Epi::Pre p;
            if constexpr (SP) {
#pragma unroll
              for (int k = 0; k < KP; ++k) set_pre(p, k, my_pre[(k * VPT + v) * TPI]);
            } else {
              p = pre[v];
            }
            if constexpr (Epi::kOut) nw = epi.store(dst, c4, acc[v], p);
            else epi.store(dst, c4, acc[v], p);
          }
        } else {
          partials[(int64_t)dst * D4 + c4] = acc[v];
        }
      }
      if (fin) pull_store(epi, n, myp, c4, nw, D4);  // group-uniform: every lane shuffles
    }
    return item;
  };
  // Items come long-chunks-first (pl.nw == 0, dedup.cu emit_items): the
  // CTAs first take the long chunks, one per CTA at a time (long_chunk: TMA
  // staging + the fused tree), then every group takes short items. Two loops
  // keep the tree's registers out of the short-item loop, which runs spill-free.
  const int n_part = pl.counters[C_PARTIALS];
  const int n_long_items = pl.fused ? n_part : 0;
  // pl.part (long-first items): 1 = the long chunks only, 2 = the short items only
  const int it_lo = pl.part == 2 ? n_part : n_long_items;
  const int it_hi = pl.part == 1 ? n_part : n_items;
  if (n_long_items > (int)blockIdx.x) {  // CTA-uniform
    if (threadIdx.x == 0) mbar_init(&s_bar, 1);
    __syncthreads();
    uint32_t parity = 0;
#pragma unroll 1
    for (int lit = blockIdx.x; lit < n_long_items; lit += gridDim.x)
      parity = long_chunk<(TPI * VPT + 255) / 256>(pl, vals, epi, lit, s_stage, &s_bar, parity, s_bc);
    __syncthreads();  // s_buf becomes s_pre
  }
  const int stride = gridDim.x * GPB;
#pragma unroll 1
  for (int it = it_lo + blockIdx.x * GPB + threadIdx.x / TPI; it < it_hi; it += stride)
    process(it);
  HP_SPAN_END(span_id);
}

// ((0 + r0) + r1) + ... over n <= HP_CHUNK rows of stride D4: all HP_CHUNK
// loads in flight (one round trip per tree level).
static __device__ __noinline__ float4 seq_sum_rows(const float4* src, int n, int D4) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 x[HP_CHUNK];
#pragma unroll
  for (int j = 0; j < HP_CHUNK; ++j)
    if (j < n) x[j] = src[(int64_t)j * D4];
#pragma unroll
  for (int j = 0; j < HP_CHUNK; ++j)
    if (j < n) acc = f4_add(acc, x[j]);
  return acc;
}

// The same sum with HP_CHUNK / 2 loads in flight (two round trips), for the
// register-capped k_combine variant (hp_debug_set_comb_lite).
static __device__ __noinline__ float4 seq_sum_rows_half(const float4* src, int n, int D4) {
  constexpr int H = HP_CHUNK / 2;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int j0 = 0; j0 < n; j0 += H) {
    float4 x[H];
#pragma unroll
    for (int j = 0; j < H; ++j)
      if (j0 + j < n) x[j] = src[(int64_t)(j0 + j) * D4];
#pragma unroll
    for (int j = 0; j < H; ++j)
      if (j0 + j < n) acc = f4_add(acc, x[j]);
  }
  return acc;
}

template <bool LITE>
__device__ __forceinline__ float4 comb_sum(const float4* src, int n, int D4) {
  if constexpr (LITE) return seq_sum_rows_half(src, n, D4);
  else return seq_sum_rows(src, n, D4);
}

// Upper levels for segments longer than HP_CHUNK: one CTA per long segment
// {partial slot, n0, dst, u}. Latency-bound (a chain per hot id), so:
//  * the CTA's first descriptor is loaded with the segment count (capacity
//    T/C + 2 entries, so the speculative read is in bounds);
//  * the epilogue's table rows (thread c4's column) are loaded before the tree;
//  * for n0 <= HP_CHUNK^2 partials (L <= 4096 rows) one level of group sums
//    goes to shared memory and the final level reads it from there.
// Same tree as before: groups of HP_CHUNK partials summed sequentially from
// +0, then the group sums sequentially (oracle.grouped_tree_sum).
constexpr int CMB_D4 = 256;  // widest row (float4) of the shared-memory path
constexpr int CMB_NT = 512;  // threads per long segment: one pass over <= 4 groups at D = 512
// One long segment, by the whole CTA: its partial rows (k_reduce's level-0
// chunk sums) summed up the tree in order, then the epilogue (apply) stores
// the result. Ends with a __syncthreads.
template <class Epi, bool LITE = false>
__device__ __forceinline__ void combine_segment(const DedupPlan& pl, const Epi& epi, int4 d,
                                                float4* s_grp) {
  const int D4 = pl.D >> 2;
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  int n = d.y;
  float4* Pp = partials + (int64_t)d.x * D4;
  constexpr int PV = (CMB_D4 + CMB_NT - 1) / CMB_NT;  // epilogue columns per thread (fast path)
  typename Epi::Pre pre[PV];
  const bool fast = n <= HP_CHUNK * HP_CHUNK && D4 <= CMB_D4;
  if (fast) {
#pragma unroll
    for (int v = 0; v < PV; ++v) {
      const int c4 = threadIdx.x + v * CMB_NT;
      if (c4 < D4 && d.z >= 0) pre[v] = epi.load(d.z, c4);
    }
    const int ng = (n + HP_CHUNK - 1) / HP_CHUNK;
    if (ng > 1) {
#pragma unroll 1
      for (int unit = threadIdx.x; unit < ng * D4; unit += blockDim.x) {
        const int g = unit / D4, c4 = unit - g * D4;
        const int e = min(HP_CHUNK, n - g * HP_CHUNK);
        s_grp[g * D4 + c4] = comb_sum<LITE>(Pp + (int64_t)g * HP_CHUNK * D4 + c4, e, D4);
      }
      __syncthreads();
    }
#pragma unroll
    for (int v = 0; v < PV; ++v) {
      const int c4 = threadIdx.x + v * CMB_NT;
      if (c4 >= D4) continue;
      float4 acc;
      if (ng > 1) {
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int g = 0; g < ng; ++g) acc = f4_add(acc, s_grp[g * D4 + c4]);
      } else {
        acc = comb_sum<LITE>(Pp + c4, n, D4);
      }
      if (d.z >= 0) epi.store(d.z, c4, acc, pre[v]);
    }
    __syncthreads();
    return;
  }
#pragma unroll 1
  while (n > HP_CHUNK) {
    const int ng = (n + HP_CHUNK - 1) / HP_CHUNK;
    const int units = ng * D4;
#pragma unroll 1
    for (int ub = 0; ub < units; ub += blockDim.x) {
      const int unit = ub + threadIdx.x;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      int g = 0, c4 = 0;
      if (unit < units) {
        g = unit / D4;
        c4 = unit - g * D4;
        const int e = min(HP_CHUNK, n - g * HP_CHUNK);
        acc = comb_sum<LITE>(Pp + (int64_t)g * HP_CHUNK * D4 + c4, e, D4);
      }
      __syncthreads();
      if (unit < units) Pp[(int64_t)g * D4 + c4] = acc;
      __syncthreads();
    }
    n = ng;
  }
#pragma unroll 1
  for (int c4 = threadIdx.x; c4 < D4; c4 += blockDim.x) {
    typename Epi::Pre p{};
    if (d.z >= 0) p = epi.load(d.z, c4);
    const float4 acc = comb_sum<LITE>(Pp + c4, n, D4);
    if (d.z >= 0) epi.store(d.z, c4, acc, p);
  }
  __syncthreads();
}

template <class Epi, bool LITE = false>
__global__ void __launch_bounds__(CMB_NT, LITE ? 2 : 1) k_combine(DedupPlan pl, Epi epi) {
  extern __shared__ __align__(16) float4 s_grp[];  // [HP_CHUNK][D4] group sums
  HP_ENTRY(SP_COMBINE);
  const int n_long = pl.counters[C_LONG];
  // (speculative read guarded by the capacity, T/16 + 2 descriptors)
  const int4 d_first = (int64_t)blockIdx.x < pl.T / HP_CHUNK + 2 ? pl.longs[blockIdx.x]
                                                                   : make_int4(0, 0, 0, 0);
#pragma unroll 1
  for (int li = blockIdx.x; li < n_long; li += gridDim.x)
    combine_segment<Epi, LITE>(pl, epi, li == (int)blockIdx.x ? d_first : pl.longs[li], s_grp);
  HP_SPAN_END(SP_COMBINE);
}

// n = 1 apply with the pull (the split apply's long chain): the long
// segments' roots AND the copy of their updated rows to every position, in
// ONE kernel. Work items come from a queue in order: first the n_long roots
// (combine + apply, then a release flag per segment), then the long chunks
// (wait for the segment's flag, copy its slab row to the chunk's <= 16
// positions). A CTA only waits on a root an earlier ticket handed to a
// running CTA: no deadlock at any residency. The queue / done counters and
// the generation word are the plan's spare counters (zeroed with the plan);
// the last CTA resets the queue and bumps the generation, so a plan may be
// applied again.
template <class Epi>
__global__ void __launch_bounds__(CMB_NT) k_combine_bcast(DedupPlan pl, Epi epi) {
  extern __shared__ __align__(16) float4 s_grp[];
  __shared__ int s_item;
  HP_ENTRY(SP_COMBINE);
  const int D4 = pl.D >> 2;
  const int n_long = pl.counters[C_LONG];
  const int n_items = n_long + pl.counters[C_PARTIALS];
  const int gen = *reinterpret_cast<volatile int*>(&pl.counters[C_GEN]) + 1;
  int* queue = &pl.counters[C_QUEUE];
#pragma unroll 1
  while (true) {
    if (threadIdx.x == 0) s_item = atomicAdd(queue, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= n_items) break;
    if (it < n_long) {
      combine_segment(pl, epi, pl.longs[it], s_grp);
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(pl.long_flag + it), "r"(gen)
                     : "memory");
      }
      continue;
    }
    const int4 c = pl.part_desc[it - n_long];  // {first sorted row, rows, dst, long index}
    if (threadIdx.x == 0 && c.z >= 0) {
      int v;
      do {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(pl.long_flag + c.w)
                     : "memory");
      } while (v != gen);
      __threadfence();
    }
    __syncthreads();
    // column q of rows r0, r0 + rs, ... (one row per CMB_NT / D4 thread slice)
    if (D4 <= CMB_NT) {
      const int q = threadIdx.x % D4, r0 = threadIdx.x / D4, rs = CMB_NT / D4;
      if (r0 < rs) {
        const float4 row =
            c.z >= 0 ? epi.w[(int64_t)c.z * D4 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = r0; r < c.y; r += rs)
          epi.out[(int64_t)pl.sorted_pos[c.x + r] * D4 + q] = row;
      }
    } else {
      for (int r = 0; r < c.y; ++r) {
        const int64_t pos = pl.sorted_pos[c.x + r];
        for (int cc = threadIdx.x; cc < D4; cc += CMB_NT)
          epi.out[pos * D4 + cc] =
              c.z >= 0 ? epi.w[(int64_t)c.z * D4 + cc] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&pl.counters[C_DONE], 1) == (int)gridDim.x - 1) {
      pl.counters[C_QUEUE] = 0;
      pl.counters[C_DONE] = 0;
      pl.counters[C_GEN] = gen;
    }
  }
  HP_SPAN_END(SP_COMBINE);
}

// Publication after a peer-store reduce (one block, launched after k_combine):
// the system-scope fence is cumulative over every store the previous kernels
// of this stream made, then the epilogue publishes (flags / counts).
template <class Epi>
__global__ void k_publish(Epi epi) {
  HP_ENTRY(SP_PUBLISH);
  __threadfence_system();
  epi.grid_done();
  HP_SPAN_END(SP_PUBLISH);
}

// ------------------------------------------------------------------ row stream

enum { RS_FIRST = 1, RS_PRE = 2, RS_END = 4, RS_FIN = 8 };

// Level 0 of the summation tree as a per-warp row stream. Warp w walks the
// items that start in its slice of sorted rows (plan bounds wb_*); each item
// becomes n gradient-row elements followed by the epilogue's kPre table rows.
// Every element is one row copied global -> shared with cp.async (each lane
// copies and later reads only its own VPT float4 columns, so no cross-lane
// smem sync is needed), F = S - kPre elements in flight, so a warp keeps F
// rows (F*D*4 bytes) of loads outstanding regardless of how the rows group
// into items, and no registers are held by in-flight loads. Positions and
// item descriptors are read 32 at a time (coalesced) one batch ahead. The sum
// is the same ((0 + r0) + r1) + ... in sorted order as k_reduce.
template <int VPT, int S, class Epi>
__global__ void __launch_bounds__(128) k_rowstream(DedupPlan pl, const float* __restrict__ vals_f,
                                                   Epi epi) {
  constexpr int D4 = VPT * 32;
  constexpr int F = S - Epi::kPre;
  static_assert(F >= 2, "row stream needs >= 2 rows in flight");
  extern __shared__ __align__(16) float4 s_rows[];  // [4 warps][S][D4]
  __shared__ int2 s_meta[4][S];
  const float4* __restrict__ vals = reinterpret_cast<const float4*>(vals_f);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * 4 + wid;
  const int T = (int)pl.T;
  const int R = (T + pl.nw - 1) / pl.nw;
  HP_ENTRY(SP_REDUCE);
  float4* ring = s_rows + (size_t)wid * S * D4;
  int ib = 0, ie = 0, rb = 0, re = 0;
  if ((int64_t)gw * R < T) {
    ib = pl.wb_item[gw];
    rb = pl.wb_row[gw];
    if ((int64_t)(gw + 1) * R >= T) {
      ie = pl.counters[C_ITEMS];
      re = T;
    } else {
      ie = pl.wb_item[gw + 1];
      re = pl.wb_row[gw + 1];
    }
  }
  // descriptor / position batches (lane l holds entry base + l), next batch prefetched
  int dbase = ib, pbase = rb;
  int4 dcur = make_int4(0, 0, 0, 0), dnxt = dcur;
  int pcur = 0, pnxt = 0;
  if (ib + lane < ie) dcur = pl.items[ib + lane];
  if (ib + 32 + lane < ie) dnxt = pl.items[ib + 32 + lane];
  if (rb + lane < re) pcur = pl.sorted_pos[rb + lane];
  if (rb + 32 + lane < re) pnxt = pl.sorted_pos[rb + 32 + lane];
  // producer cursor: item pi, element pj of pn + pnpre
  int pi = ib, pj = 0, pn = 0, pdst = 0, pfin = 0, pnpre = 0, gp = rb;
  auto fetch_item = [&]() {
    if (pi - dbase == 32) {
      dcur = dnxt;
      dbase += 32;
      if (dbase + 32 + lane < ie) dnxt = pl.items[dbase + 32 + lane];
    }
    const int k = pi - dbase;
    pn = __shfl_sync(0xffffffffu, dcur.y, k);
    pdst = __shfl_sync(0xffffffffu, dcur.z, k);
    pfin = __shfl_sync(0xffffffffu, dcur.w, k) > 0;  // < 0: chunk of a long segment
    pnpre = (pfin && pdst >= 0) ? Epi::kPre : 0;
  };
  if (pi < ie) fetch_item();
  auto issue = [&](int e) {
    const int slot = e % S;
    const float4* src;
    int flags;
    if (pj < pn) {
      if (gp - pbase == 32) {
        pcur = pnxt;
        pbase += 32;
        if (pbase + 32 + lane < re) pnxt = pl.sorted_pos[pbase + 32 + lane];
      }
      const int pos = __shfl_sync(0xffffffffu, pcur, gp - pbase);
      ++gp;
      src = vals + (int64_t)pos * D4;
      flags = pj == 0 ? RS_FIRST : 0;
    } else {
      src = epi.pre_row(pj - pn, pdst);
      flags = RS_PRE;
    }
    float4* dstp = ring + slot * D4;
#pragma unroll
    for (int v = 0; v < VPT; ++v) cp_async16(dstp + lane + v * 32, src + lane + v * 32);
    const bool end = pj + 1 == pn + pnpre;
    if (lane == 0)
      s_meta[wid][slot] = make_int2(pdst, flags | (end ? RS_END : 0) | (pfin ? RS_FIN : 0) |
                                              (pnpre << 8));
    if (end) {
      ++pi;
      pj = 0;
      if (pi < ie) fetch_item();
    } else {
      ++pj;
    }
  };
  int issued = 0;
#pragma unroll 1
  for (int s = 0; s < F; ++s) {
    if (pi < ie) issue(issued++);
    cp_async_commit();
  }
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  float4 acc[VPT];
#pragma unroll
  for (int v = 0; v < VPT; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
  for (int m = 0; m < issued; ++m) {
    cp_async_wait<F - 1>();
    __syncwarp();
    const int slot = m % S;
    const int2 mt = s_meta[wid][slot];
    const float4* row = ring + slot * D4;
    if (!(mt.y & RS_PRE)) {
      const bool first = mt.y & RS_FIRST;
#pragma unroll
      for (int v = 0; v < VPT; ++v) {
        const float4 x = row[lane + v * 32];
        acc[v] = f4_add(first ? make_float4(0.f, 0.f, 0.f, 0.f) : acc[v], x);
      }
    }
    if (mt.y & RS_END) {
      const int dst = mt.x;
      if (!(mt.y & RS_FIN)) {
#pragma unroll
        for (int v = 0; v < VPT; ++v) partials[(int64_t)dst * D4 + lane + v * 32] = acc[v];
      } else if (dst >= 0) {
        const int npre = mt.y >> 8;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
          const int c4 = lane + v * 32;
          typename Epi::Pre pre;
          if constexpr (Epi::kPre > 0) {
#pragma unroll
            for (int k = 0; k < Epi::kPre; ++k)
              set_pre(pre, k, ring[((m - npre + 1 + k + S) % S) * D4 + c4]);
          } else {
            pre = epi.load(dst, c4);
          }
          epi.store(dst, c4, acc[v], pre);
        }
      }
    }
    __syncwarp();
    if (pi < ie) issue(issued++);
    cp_async_commit();
  }
  cp_async_wait<0>();
  HP_SPAN_END(SP_REDUCE);
}

template <int VPT, class Epi>
void launch_rowstream(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st) {
  constexpr int S = VPT == 1 ? 16 : (VPT == 2 ? 12 : (VPT == 4 ? 8 : 6));
  constexpr size_t smem = (size_t)4 * S * VPT * 32 * sizeof(float4);
  auto kern = k_rowstream<VPT, S, Epi>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  launch_k(kern, dim3(pl.nw / 4), dim3(128), smem, st, pl, vals, epi);
}

template <int TPI, int VPT, int B, class Epi>
void launch_k_reduce_b(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st,
                       int blocks) {
  launch_k(k_reduce<TPI, VPT, B, Epi>, dim3(blocks), dim3(256), 0, st, pl, vals, epi);
}

template <int TPI, int VPT, class Epi>
void launch_k_reduce(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st) {
  // rows in flight per batch: most items hold 1-2 rows, so a small batch keeps
  // registers (and so resident items per SM) up without costing the hot chunks much
  // measured: B=2 beats 4 and 8 at VPT=2; B=4 at VPT=1 (D <= 128)
  // keeps the default variant spill-free (B=8 spilled 16-52 B)
  constexpr int B = VPT >= 2 ? 2 : 4;
  // <= one group per item, many waves (each block fences once if its epilogue
  // stores to peers; hp_debug_set_owner_waves(0) keeps those in one resident wave)
  const int blocks = grid_for(pl.part == 1 ? 2 * pl.T / HP_CHUNK + 2 : pl.T, 256 / TPI,
                              sm_count() * (Epi::kRemote && !g_owner_waves ? 3 : g_reduce_bps));
  if (VPT == 2 && g_reduce_b == 4)
    launch_k_reduce_b<TPI, VPT, 4>(pl, vals, epi, st, blocks);
  else if (VPT == 2 && g_reduce_b == 8)
    launch_k_reduce_b<TPI, VPT, 8>(pl, vals, epi, st, blocks);
  else
    launch_k_reduce_b<TPI, VPT, B>(pl, vals, epi, st, blocks);
}

// The long segments' chunks alone on TMA (pl.part == 1, hp_debug_set_long_tma):
// one CTA per chunk at a time, its <= 16 gradient rows bulk-copied into shared
// memory (cta_stage_sum: batches of stage_rows(D) rows, one elected lane per
// row) and summed per column in row order from +0.0 -> the chunk's partial
// slot. Two DRAM round trips per 16-row chunk at D = 512 instead of eight.
template <int CPT>
__global__ void __launch_bounds__(256)
k_reduce_long_tma(DedupPlan pl, const float* __restrict__ vals_f) {
  __shared__ __align__(128) float4 s_stage[STAGE_F4];
  __shared__ uint64_t s_bar;
  HP_ENTRY(SP_REDUCE);
  const float4* vals = reinterpret_cast<const float4*>(vals_f);
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  const int D4 = pl.D >> 2, SR = stage_rows(pl.D);
  const int n_part = pl.counters[C_PARTIALS];
  if (threadIdx.x == 0) mbar_init(&s_bar, 1);
  __syncthreads();
  uint32_t parity = 0;
#pragma unroll 1
  for (int it = blockIdx.x; it < n_part; it += gridDim.x) {  // long-first: [0, n_part) are chunks
    const int4 item = pl.items[it];
    parity = cta_stage_sum<CPT>(
        s_stage, &s_bar, parity, item.y, D4, SR,
        [&](int j) { return vals + (int64_t)pl.sorted_pos[item.x + j] * D4; },
        [&](int, int c4, float4 a) { partials[(int64_t)item.z * D4 + c4] = a; }, false);
    __syncthreads();  // s_stage is reused by the next chunk
  }
  HP_SPAN_END(SP_REDUCE);
}

inline void launch_k_reduce_long_tma(const DedupPlan& pl, const float* vals, cudaStream_t st) {
  const int D4 = pl.D >> 2;
  const int g = grid_for(2 * pl.T / HP_CHUNK + 2, 1, sm_count() * std::max(1, g_long_tma));
  if (D4 <= 256) launch_k(k_reduce_long_tma<1>, dim3(g), dim3(256), 0, st, pl, vals);
  else if (D4 <= 512) launch_k(k_reduce_long_tma<2>, dim3(g), dim3(256), 0, st, pl, vals);
  else launch_k(k_reduce_long_tma<4>, dim3(g), dim3(256), 0, st, pl, vals);
}

// The long segments' chunks alone (pl.part == 1, hp_debug_set_long_b8 > 0;
// A/B, off by default: faster alone, slower in the step, see the header):
// every item is a full 16-row chunk, so each group keeps 8 rows in flight (2
// round trips per chunk instead of 8) on one float4 column per thread. Long chunks only write partial rows, so no epilogue is
// compiled in (EpiSend, never called): one instantiation per width, spill-free.
inline void launch_k_reduce_long(const DedupPlan& pl, const float* vals, cudaStream_t st) {
  const int D4 = pl.D >> 2;
  const EpiSend epi{nullptr, D4};
  // the chunk count is on the device: at most one block per SM (g_long_b8
  // blocks per SM when > 1), grid-striding over the chunks
  const int64_t items = 2 * pl.T / HP_CHUNK + 2;
  const int cap = sm_count() * std::max(1, g_long_b8);
  if (D4 <= 32) launch_k_reduce_b<32, 1, 8>(pl, vals, epi, st, grid_for(items, 8, cap));
  else if (D4 <= 64) launch_k_reduce_b<64, 1, 8>(pl, vals, epi, st, grid_for(items, 4, cap));
  else if (D4 <= 128) launch_k_reduce_b<128, 1, 8>(pl, vals, epi, st, grid_for(items, 2, cap));
  else if (D4 <= 256) launch_k_reduce_b<256, 1, 8>(pl, vals, epi, st, grid_for(items, 1, cap));
  else launch_k_reduce_b<256, 2, 4>(pl, vals, epi, st, grid_for(items, 1, cap));
}

template <class Epi>
int launch_reduce(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st) {
  if (pl.T == 0) return HP_OK;
  const int D4 = pl.D >> 2;
  if (pl.nw > 0 && rs_stages(pl.D) > 0 && !g_rowstream_off) {
    switch (D4) {
      case 32: launch_rowstream<1>(pl, vals, epi, st); break;
      case 64: launch_rowstream<2>(pl, vals, epi, st); break;
      case 128: launch_rowstream<4>(pl, vals, epi, st); break;
      default: launch_rowstream<8>(pl, vals, epi, st); break;
    }
    HP_LAUNCHED(1, "k_rowstream");
  } else if (pl.part == 1 && g_long_tma && pl.reorder && pl.D <= 4 * 4096) {
    launch_k_reduce_long_tma(pl, vals, st);
    HP_LAUNCHED(1, "k_reduce_long_tma");
  } else if (pl.part == 1 && g_long_b8) {
    launch_k_reduce_long(pl, vals, st);
    HP_LAUNCHED(1, "k_reduce (long chunks)");
  } else {
    if (D4 <= 32) launch_k_reduce<32, 1>(pl, vals, epi, st);
    else if (D4 <= 64) launch_k_reduce<32, 2>(pl, vals, epi, st);
    else if (D4 <= 128) launch_k_reduce<64, 2>(pl, vals, epi, st);
    // wide rows (NMT D = 1024, D = 2048): wider groups at 2 float4 columns per
    // thread keep the kernel spill-free (4 columns spilled 300-700 B per thread)
    else if (D4 <= 256) launch_k_reduce<128, 2>(pl, vals, epi, st);
    else launch_k_reduce<256, 2>(pl, vals, epi, st);
    HP_LAUNCHED(1, "k_reduce");
  }
  if (pl.part == 2) return HP_OK;  // short items only: no long segment to close (nor publish)
  // fused tree (items in long-first order, pl.nw == 0): k_reduce closed every
  // long segment itself (long_chunk); otherwise one CTA per long segment
  if (pl.fused) {
    if constexpr (Epi::kRemote) {
      launch_k(k_publish<Epi>, dim3(1), dim3(64), 0, st, epi);
      HP_LAUNCHED(1, "k_publish");
    }
    return HP_OK;
  }
  // hp_debug_set_combine_blocks caps the k_combine grid for peer epilogues
  const int cblocks = grid_for(pl.T / (HP_CHUNK + 1) + 1, 1,
                               Epi::kRemote && g_combine_blocks > 0 ? g_combine_blocks : sm_count());
  const size_t csmem = (size_t)HP_CHUNK * std::min(D4, CMB_D4) * sizeof(float4);
  static bool cconf = false;
  if (!cconf) {
    HP_CUDA(cudaFuncSetAttribute(k_combine<Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((size_t)HP_CHUNK * CMB_D4 * sizeof(float4))));
    cconf = true;
  }
  if constexpr (Epi::kOut && !Epi::kRemote) {
    if (pl.part == 1 && pl.cbcast) {  // roots + the pull of their rows, one work queue
      static bool bconf = false;
      if (!bconf) {
        HP_CUDA(cudaFuncSetAttribute(k_combine_bcast<Epi>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)((size_t)HP_CHUNK * CMB_D4 * sizeof(float4))));
        bconf = true;
      }
      // a fraction of the SMs (one 512-thread CTA fills an SM's registers): the
      // short items' k_reduce runs beside it on the rest
      const int g = pl.cbcast > 1 ? pl.cbcast : std::max(1, sm_count() / 3);
      launch_k(k_combine_bcast<Epi>, dim3(g), dim3(CMB_NT), csmem, st, pl, epi);
      HP_LAUNCHED(1, "k_combine_bcast");
      return HP_OK;
    }
  }
  if (g_comb_lite) {  // A/B: 64 registers, two CTAs per SM
    static bool lconf = false;
    if (!lconf) {
      HP_CUDA(cudaFuncSetAttribute(k_combine<Epi, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)((size_t)HP_CHUNK * CMB_D4 * sizeof(float4))));
      lconf = true;
    }
    launch_k(k_combine<Epi, true>, dim3(cblocks), dim3(CMB_NT), csmem, st, pl, epi);
  } else {
    launch_k(k_combine<Epi>, dim3(cblocks), dim3(CMB_NT), csmem, st, pl, epi);
  }
  HP_LAUNCHED(1, "k_combine");
  if (pl.part == 1) return HP_OK;  // split push: the caller publishes after the join
  if constexpr (Epi::kRemote) {
    launch_k(k_publish<Epi>, dim3(1), dim3(64), 0, st, epi);
    HP_LAUNCHED(1, "k_publish");
  }
  return HP_OK;
}

}  // namespace hp
