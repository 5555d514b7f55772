// Segmented row reduction over a DedupPlan, with fused epilogues:
//   EpiSend   -> summed row written to its send slot           (K1 values half)
//   EpiApply  -> merged gradient scaled + optimizer row update  (K4 scatter-apply)
//
// Summation tree (oracle.tree_sum): each segment's rows, in ascending sorted
// position, are summed sequentially in groups of HP_CHUNK; while more than
// HP_CHUNK partials remain they are grouped again. Level 0 runs one warp per
// (segment, chunk) item over the whole grid (hot ids spread across SMs);
// upper levels of long segments run one CTA per segment (k_combine).
// Every add / mul / div / sqrt is an explicit round-to-nearest intrinsic so
// the result is bit-identical to the numpy oracle.
//
// Reference: server aggregation + update (sparseplan/simulate.py:294-323,
// 358-367); one update per (Weight, partition) per step.
#include "hp_dedup.cuh"

namespace hp {
namespace {

// Epilogue interface: Pre load(dst, c4) is issued BEFORE the row loads (it
// only depends on the item), store(dst, c4, g, pre) consumes the summed float4.
struct EpiSend {
  float4* rows;
  int D4;
  struct Pre {};
  __device__ __forceinline__ Pre load(int, int) const { return {}; }
  __device__ __forceinline__ void store(int dst, int c4, float4 g, Pre) const {
    rows[(int64_t)dst * D4 + c4] = g;
  }
};

template <int OPT>
struct EpiApply {
  float4* w;
  float4* s0;
  float4* s1;
  hp_optim o;
  int D4;
  struct Pre {
    float4 w, a, b;
  };

  __device__ __forceinline__ Pre load(int dst, int c4) const {
    Pre p;
    const int64_t off = (int64_t)dst * D4 + c4;
    p.w = w[off];
    p.a = p.b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (OPT != HP_OPT_SGD) p.a = s0[off];
    if (OPT == HP_OPT_ADAM) p.b = s1[off];
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
      wv = __fsub_rn(wv, __fdiv_rn(__fmul_rn(o.lr_t, a), __fadd_rn(__fsqrt_rn(b), o.eps)));
    }
  }

  __device__ __forceinline__ void store(int dst, int c4, float4 g, Pre p) const {
    upd(p.w.x, p.a.x, p.b.x, g.x);
    upd(p.w.y, p.a.y, p.b.y, g.y);
    upd(p.w.z, p.a.z, p.b.z, g.z);
    upd(p.w.w, p.a.w, p.b.w, g.w);
    const int64_t off = (int64_t)dst * D4 + c4;
    w[off] = p.w;
    if (OPT != HP_OPT_SGD) s0[off] = p.a;
    if (OPT == HP_OPT_ADAM) s1[off] = p.b;
  }
};

// Level 0 of the summation tree. A group of TPI threads owns an item
// {j0, n <= HP_CHUNK, dst, final}; each thread owns VPT float4 columns
// (c4 = lane-in-group + k*TPI). Row positions are loaded once per warp and
// broadcast by shuffle; B rows x VPT columns are in flight per thread before
// the in-order fp32 adds. Final items run the epilogue (its table-row loads
// are issued together with the positions); long-segment chunks write a
// partial row for k_combine. Small groups + <= 64 registers keep many items
// in flight per SM: the kernel is latency-bound on the item chain
// (descriptor -> positions/table rows -> gradient rows).
template <int TPI, int VPT, int B, class Epi>
__global__ void __launch_bounds__(256, 3)
k_reduce(DedupPlan pl, const float* __restrict__ vals_f, Epi epi) {
  const float4* __restrict__ vals = reinterpret_cast<const float4*>(vals_f);
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  const int D4 = pl.D >> 2;
  constexpr int GPB = 256 / TPI;
  const int q = threadIdx.x % TPI;
  const int lane = threadIdx.x & 31;
  const int n_items = pl.counters[C_ITEMS];
  for (int it = blockIdx.x * GPB + threadIdx.x / TPI; it < n_items; it += gridDim.x * GPB) {
    const int4 item = pl.items[it];
    const int j0 = item.x, n = item.y, dst = item.z;
    const bool fin = item.w != 0;
    typename Epi::Pre pre[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v)
      if (fin && dst >= 0 && q + v * TPI < D4) pre[v] = epi.load(dst, q + v * TPI);
    const int myp = lane < n ? pl.sorted_pos[j0 + lane] : 0;
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
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      const int c4 = q + v * TPI;
      if (c4 >= D4) continue;
      if (fin) {
        if (dst >= 0) epi.store(dst, c4, acc[v], pre[v]);
      } else {
        partials[(int64_t)dst * D4 + c4] = acc[v];
      }
    }
  }
}

// ((0 + r0) + r1) + ... over n <= HP_CHUNK rows of stride D4, 8 loads in flight.
__device__ __forceinline__ float4 seq_sum_rows(const float4* src, int n, int D4) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j0 = 0; j0 < n; j0 += 8) {
    float4 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j0 + j < n) x[j] = src[(int64_t)(j0 + j) * D4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j0 + j < n) acc = f4_add(acc, x[j]);
  }
  return acc;
}

// Upper levels for segments longer than HP_CHUNK: one CTA per long segment
// {partial slot, n0, dst, u}, in place over its partial rows.
template <class Epi>
__global__ void __launch_bounds__(256) k_combine(DedupPlan pl, Epi epi) {
  const int D4 = pl.D >> 2;
  const int n_long = pl.counters[C_LONG];
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  for (int li = blockIdx.x; li < n_long; li += gridDim.x) {
    const int4 d = pl.longs[li];
    int n = d.y;
    float4* Pp = partials + (int64_t)d.x * D4;
    while (n > HP_CHUNK) {
      const int ng = (n + HP_CHUNK - 1) / HP_CHUNK;
      const int units = ng * D4;
      for (int ub = 0; ub < units; ub += blockDim.x) {
        const int unit = ub + threadIdx.x;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int g = 0, c4 = 0;
        if (unit < units) {
          g = unit / D4;
          c4 = unit - g * D4;
          const int e = min(HP_CHUNK, n - g * HP_CHUNK);
          acc = seq_sum_rows(Pp + (int64_t)g * HP_CHUNK * D4 + c4, e, D4);
        }
        __syncthreads();
        if (unit < units) Pp[(int64_t)g * D4 + c4] = acc;
        __syncthreads();
      }
      n = ng;
    }
    for (int c4 = threadIdx.x; c4 < D4; c4 += blockDim.x) {
      typename Epi::Pre pre{};
      if (d.z >= 0) pre = epi.load(d.z, c4);
      const float4 acc = seq_sum_rows(Pp + c4, n, D4);
      if (d.z >= 0) epi.store(d.z, c4, acc, pre);
    }
    __syncthreads();
  }
}

template <int TPI, int VPT, class Epi>
void launch_k_reduce(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st) {
  constexpr int B = VPT >= 8 ? 1 : 8 / VPT;
  const int blocks = grid_for(pl.T, 256 / TPI, sm_count() * 16);  // <= one group per item
  k_reduce<TPI, VPT, B, Epi><<<blocks, 256, 0, st>>>(pl, vals, epi);
}

template <class Epi>
int launch_reduce(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st) {
  if (pl.T == 0) return HP_OK;
  const int D4 = pl.D >> 2;
  if (D4 <= 32) launch_k_reduce<32, 1>(pl, vals, epi, st);
  else if (D4 <= 64) launch_k_reduce<32, 2>(pl, vals, epi, st);
  else if (D4 <= 128) launch_k_reduce<64, 2>(pl, vals, epi, st);
  else if (D4 <= 256) launch_k_reduce<64, 4>(pl, vals, epi, st);
  else launch_k_reduce<128, 4>(pl, vals, epi, st);
  HP_LAUNCHED(1, "k_reduce");
  const int cblocks = grid_for(pl.T / HP_CHUNK + 1, 1, sm_count() * 2);
  k_combine<Epi><<<cblocks, 256, 0, st>>>(pl, epi);
  HP_LAUNCHED(1, "k_combine");
  return HP_OK;
}

int check_slab(const hp_slab& s, int opt) {
  HP_REQUIRE(s.w != nullptr && s.part_base != nullptr, "slab.w / slab.part_base is NULL");
  HP_REQUIRE(s.D >= 4 && s.D % 4 == 0 && s.D <= 2048, "D must be a multiple of 4 in [4, 2048]");
  HP_REQUIRE(opt == HP_OPT_SGD || s.s0 != nullptr, "optimizer state s0 is NULL");
  HP_REQUIRE(opt != HP_OPT_ADAM || s.s1 != nullptr, "Adam state s1 is NULL");
  HP_REQUIRE(opt >= HP_OPT_SGD && opt <= HP_OPT_ADAM, "unknown optimizer kind");
  return HP_OK;
}

template <int OPT>
EpiApply<OPT> make_apply(const hp_slab& s, const hp_optim& o) {
  EpiApply<OPT> e{reinterpret_cast<float4*>(s.w), reinterpret_cast<float4*>(s.s0),
                  reinterpret_cast<float4*>(s.s1), o, s.D >> 2};
  return e;
}

int apply_plan(const DedupPlan& pl, const float* vals, const hp_slab& s, const hp_optim& o,
               cudaStream_t st) {
  switch (o.kind) {
    case HP_OPT_SGD: return launch_reduce(pl, vals, make_apply<HP_OPT_SGD>(s, o), st);
    case HP_OPT_ADAGRAD: return launch_reduce(pl, vals, make_apply<HP_OPT_ADAGRAD>(s, o), st);
    default: return launch_reduce(pl, vals, make_apply<HP_OPT_ADAM>(s, o), st);
  }
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" {

size_t hp_dedup_ws_bytes(int64_t T, int32_t D, int32_t P, int32_t nranks) {
  (void)nranks;
  return dedup_ws_bytes(T, D, P);
}

int hp_dedup_plan(const int64_t* ids, int64_t T, int32_t D, int64_t V, int32_t P,
                  const int32_t* owner, int32_t nranks, int64_t* send_ids, int32_t* counts,
                  int32_t* inv, int32_t* dest_counts, int32_t* n_uniq, void* ws,
                  size_t ws_bytes, void* stream) {
  DedupPlan pl;
  int rc = carve_plan(&pl, ws, ws_bytes, T, D, V, P, nranks);
  if (rc) return rc;
  HP_REQUIRE(T == 0 || ids != nullptr, "ids is NULL");
  HP_REQUIRE(owner != nullptr || nranks == 1, "owner table required when nranks > 1");
  return build_plan(pl, ids, owner, nullptr, send_ids, counts, inv, dest_counts, n_uniq,
                    static_cast<cudaStream_t>(stream));
}

int hp_sort_dedup_route(const int64_t* ids, const float* vals, int64_t T, int32_t D, int64_t V,
                        int32_t P, const int32_t* owner, int32_t nranks, int64_t* send_ids,
                        float* send_rows, int32_t* counts, int32_t* inv, int32_t* dest_counts,
                        int32_t* n_uniq, void* ws, size_t ws_bytes, void* stream) {
  HP_REQUIRE(D >= 4 && D % 4 == 0 && D <= 2048, "D must be a multiple of 4 in [4, 2048]");
  HP_REQUIRE(T == 0 || (vals != nullptr && send_rows != nullptr), "vals / send_rows is NULL");
  DedupPlan pl;
  int rc = carve_plan(&pl, ws, ws_bytes, T, D, V, P, nranks);
  if (rc) return rc;
  HP_REQUIRE(T == 0 || ids != nullptr, "ids is NULL");
  HP_REQUIRE(owner != nullptr || nranks == 1, "owner table required when nranks > 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = build_plan(pl, ids, owner, nullptr, send_ids, counts, inv, dest_counts, n_uniq, st);
  if (rc) return rc;
  EpiSend epi{reinterpret_cast<float4*>(send_rows), D >> 2};
  return launch_reduce(pl, vals, epi, st);
}

int hp_merge_apply(const int64_t* ids, const float* rows, int64_t R, hp_slab slab, hp_optim opt,
                   void* ws, size_t ws_bytes, void* stream) {
  int rc = check_slab(slab, opt.kind);
  if (rc) return rc;
  DedupPlan pl;
  if ((rc = carve_plan(&pl, ws, ws_bytes, R, slab.D, slab.V, slab.P, 1))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = build_plan(pl, ids, nullptr, slab.part_base, nullptr, nullptr, nullptr, nullptr,
                       nullptr, st)))
    return rc;
  return apply_plan(pl, rows, slab, opt, st);
}

int hp_apply_plan_build(const int64_t* ids, int64_t R, hp_slab slab, void* ws, size_t ws_bytes,
                        void* stream) {
  HP_REQUIRE(slab.part_base != nullptr, "slab.part_base is NULL");
  HP_REQUIRE(R == 0 || ids != nullptr, "ids is NULL");
  DedupPlan pl;
  int rc = carve_plan(&pl, ws, ws_bytes, R, slab.D, slab.V, slab.P, 1);
  if (rc) return rc;
  return build_plan(pl, ids, nullptr, slab.part_base, nullptr, nullptr, nullptr, nullptr,
                    nullptr, static_cast<cudaStream_t>(stream));
}

int hp_local_apply(const int64_t* ids, const float* vals, int64_t T, hp_slab slab, hp_optim opt,
                   void* ws, size_t ws_bytes, void* stream) {
  return hp_merge_apply(ids, vals, T, slab, opt, ws, ws_bytes, stream);
}

int hp_apply_plan(const float* rows, int64_t R, hp_slab slab, hp_optim opt, void* ws,
                  size_t ws_bytes, void* stream) {
  int rc = check_slab(slab, opt.kind);
  if (rc) return rc;
  HP_REQUIRE(R == 0 || rows != nullptr, "rows is NULL");
  DedupPlan pl;
  if ((rc = carve_plan(&pl, ws, ws_bytes, R, slab.D, slab.V, slab.P, 1))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the radix sort leaves the positions in pos[passes & 1] on the large path
  if (R > HP_SMALL_MAX) {
    const int passes = (pl.key_bits + HP_RADIX_BITS - 1) / HP_RADIX_BITS;
    pl.sorted_pos = pl.pos[passes & 1];
  }
  return apply_plan(pl, rows, slab, opt, st);
}

// Error word of the last plan built in ws (bit 0: id out of range, bit 1: row
// not homed on this rank). Synchronises the stream.
int hp_plan_status(const void* ws, int32_t* out_err, void* stream) {
  HP_REQUIRE(ws != nullptr && out_err != nullptr, "NULL argument");
  const int32_t* counters = static_cast<const int32_t*>(ws);  // carved first
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_CUDA(cudaMemcpyAsync(out_err, counters + C_ERR, 4, cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  return HP_OK;
}

}  // extern "C"
