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

struct EpiSend {
  float4* rows;
  const int32_t* sigma;
  int D4;
  __device__ __forceinline__ void operator()(int u, int c4, float4 g) const {
    rows[(int64_t)sigma[u] * D4 + c4] = g;
  }
};

template <int OPT>
struct EpiApply {
  float4* w;
  float4* s0;
  float4* s1;
  const int64_t* part_base;
  const uint32_t* uniq_key;
  Router route;
  hp_optim o;
  int D4;
  int* err;

  __device__ __forceinline__ float upd(float& wv, float& a, float& b, float g) const {
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
    return wv;
  }

  __device__ __forceinline__ void operator()(int u, int c4, float4 g) const {
    const int64_t id = uniq_key[u];
    const int p = route.part(id);
    const int64_t base = part_base[p];
    if (base < 0) {  // row not homed on this rank: routing bug or bad ids
      atomicOr(err, 2);
      return;
    }
    const int64_t off = (base + (id - route.lo(p))) * D4 + c4;
    float4 wv = w[off];
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
    if (OPT != HP_OPT_SGD) a = s0[off];
    if (OPT == HP_OPT_ADAM) b = s1[off];
    upd(wv.x, a.x, b.x, g.x);
    upd(wv.y, a.y, b.y, g.y);
    upd(wv.z, a.z, b.z, g.z);
    upd(wv.w, a.w, b.w, g.w);
    w[off] = wv;
    if (OPT != HP_OPT_SGD) s0[off] = a;
    if (OPT == HP_OPT_ADAM) s1[off] = b;
  }
};

// Level 0: one warp per (segment, chunk) item.
template <int VPL, class Epi>
__global__ void __launch_bounds__(256)
k_reduce(DedupPlan pl, const float* __restrict__ vals_f, Epi epi) {
  constexpr int UNR = VPL >= 8 ? 1 : 8 / VPL;
  const float4* __restrict__ vals = reinterpret_cast<const float4*>(vals_f);
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  const int D4 = pl.D >> 2;
  const int lane = threadIdx.x & 31;
  const int n_items = pl.counters[C_ITEMS];
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n_items; it += nw) {
    const int u = pl.item_seg[it];
    const int k = it - pl.item_off[u];
    const int s0 = pl.seg_start[u], s1 = pl.seg_start[u + 1];
    const int j0 = s0 + k * HP_CHUNK, j1 = min(j0 + HP_CHUNK, s1);
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int jb = j0; jb < j1; jb += 32) {
      const int nb = min(32, j1 - jb);
      const int myp = lane < nb ? pl.sorted_pos[jb + lane] : 0;
      int q = 0;
      for (; q + UNR <= nb; q += UNR) {
        float4 x[UNR][VPL];
#pragma unroll
        for (int e = 0; e < UNR; ++e) {
          const int64_t rb = (int64_t)__shfl_sync(0xffffffffu, myp, q + e) * D4;
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const int c4 = lane + 32 * v;
            if (c4 < D4) x[e][v] = ldg_stream(vals + rb + c4);
          }
        }
#pragma unroll
        for (int e = 0; e < UNR; ++e)
#pragma unroll
          for (int v = 0; v < VPL; ++v) acc[v] = f4_add(acc[v], x[e][v]);
      }
      for (; q < nb; ++q) {
        const int64_t rb = (int64_t)__shfl_sync(0xffffffffu, myp, q) * D4;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int c4 = lane + 32 * v;
          if (c4 < D4) acc[v] = f4_add(acc[v], ldg_stream(vals + rb + c4));
        }
      }
    }
    if (s1 - s0 <= HP_CHUNK) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c4 = lane + 32 * v;
        if (c4 < D4) epi(u, c4, acc[v]);
      }
    } else {
      float4* dst = partials + (int64_t)(pl.part_off[u] + k) * D4;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c4 = lane + 32 * v;
        if (c4 < D4) dst[c4] = acc[v];
      }
    }
  }
}

// Upper levels for segments longer than HP_CHUNK: one CTA per segment,
// in-place over the segment's partial rows.
template <class Epi>
__global__ void __launch_bounds__(256) k_combine(DedupPlan pl, Epi epi) {
  const int D4 = pl.D >> 2;
  const int n_long = pl.counters[C_LONG];
  float4* partials = reinterpret_cast<float4*>(pl.partials);
  for (int li = blockIdx.x; li < n_long; li += gridDim.x) {
    const int u = pl.long_list[li];
    const int L = pl.seg_start[u + 1] - pl.seg_start[u];
    int n = (L + HP_CHUNK - 1) / HP_CHUNK;
    float4* Pp = partials + (int64_t)pl.part_off[u] * D4;
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
          const float4* src = Pp + (int64_t)g * HP_CHUNK * D4 + c4;
          for (int j = 0; j < e; ++j) acc = f4_add(acc, src[(int64_t)j * D4]);
        }
        __syncthreads();
        if (unit < units) Pp[(int64_t)g * D4 + c4] = acc;
        __syncthreads();
      }
      n = ng;
    }
    for (int c4 = threadIdx.x; c4 < D4; c4 += blockDim.x) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int j = 0; j < n; ++j) acc = f4_add(acc, Pp[(int64_t)j * D4 + c4]);
      epi(u, c4, acc);
    }
    __syncthreads();
  }
}

template <class Epi>
int launch_reduce(const DedupPlan& pl, const float* vals, const Epi& epi, cudaStream_t st) {
  if (pl.T == 0) return HP_OK;
  const int D4 = pl.D >> 2;
  const int sms = sm_count();
  const int blocks = grid_for(pl.T, 8, sms * 8);  // <= one warp per item
  if (D4 <= 32)
    k_reduce<1, Epi><<<blocks, 256, 0, st>>>(pl, vals, epi);
  else if (D4 <= 64)
    k_reduce<2, Epi><<<blocks, 256, 0, st>>>(pl, vals, epi);
  else if (D4 <= 128)
    k_reduce<4, Epi><<<blocks, 256, 0, st>>>(pl, vals, epi);
  else if (D4 <= 256)
    k_reduce<8, Epi><<<blocks, 256, 0, st>>>(pl, vals, epi);
  else
    k_reduce<16, Epi><<<blocks, 256, 0, st>>>(pl, vals, epi);
  HP_LAUNCHED(1, "k_reduce");
  const int cblocks = grid_for(pl.T / HP_CHUNK + 1, 1, sms * 2);
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
EpiApply<OPT> make_apply(const DedupPlan& pl, const hp_slab& s, const hp_optim& o) {
  EpiApply<OPT> e{reinterpret_cast<float4*>(s.w), reinterpret_cast<float4*>(s.s0),
                  reinterpret_cast<float4*>(s.s1), s.part_base, pl.uniq_key,
                  Router(s.V, s.P), o, s.D >> 2, &pl.counters[C_ERR]};
  return e;
}

int apply_plan(const DedupPlan& pl, const float* vals, const hp_slab& s, const hp_optim& o,
               cudaStream_t st) {
  switch (o.kind) {
    case HP_OPT_SGD: return launch_reduce(pl, vals, make_apply<HP_OPT_SGD>(pl, s, o), st);
    case HP_OPT_ADAGRAD: return launch_reduce(pl, vals, make_apply<HP_OPT_ADAGRAD>(pl, s, o), st);
    default: return launch_reduce(pl, vals, make_apply<HP_OPT_ADAM>(pl, s, o), st);
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
  return build_plan(pl, ids, owner, send_ids, counts, inv, dest_counts, n_uniq,
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
  rc = build_plan(pl, ids, owner, send_ids, counts, inv, dest_counts, n_uniq, st);
  if (rc) return rc;
  EpiSend epi{reinterpret_cast<float4*>(send_rows), pl.sigma, D >> 2};
  return launch_reduce(pl, vals, epi, st);
}

int hp_merge_apply(const int64_t* ids, const float* rows, int64_t R, hp_slab slab, hp_optim opt,
                   void* ws, size_t ws_bytes, void* stream) {
  int rc = check_slab(slab, opt.kind);
  if (rc) return rc;
  DedupPlan pl;
  if ((rc = carve_plan(&pl, ws, ws_bytes, R, slab.D, slab.V, slab.P, 1))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((rc = build_plan(pl, ids, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, st)))
    return rc;
  return apply_plan(pl, rows, slab, opt, st);
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
