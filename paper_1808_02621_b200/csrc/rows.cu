// K5 gather, K6 stitch, table init, dense scale+cast epilogue.
//
// K5 (PS pull, sparseplan/simulate.py:195-199): out[i] = slab row of ids[i].
// K6 (stitch):                     out[t] = rows[inv[t]].
// Both are warp-per-row copies with several rows in flight per warp and
// 128-bit loads/stores; bytes moved = rows * D * 4 read + written.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "hp_dedup.cuh"

namespace hp {
namespace {

struct SrcSlab {  // row of a global id in this rank's slab (nullptr: not homed / dropped id)
  const float4* w;
  const int64_t* part_base;
  const int64_t* ids;
  Router route;
  int64_t V;
  int D4;
  __device__ __forceinline__ const float4* operator()(int64_t i) const {
    const int64_t id = ids[i];
    if (id < 0 || id >= V) return nullptr;  // out-of-range id: a zero row (never clamped)
    const int p = route.part(id);
    const int64_t b = part_base[p];
    return b < 0 ? nullptr : w + (b + (id - route.lo(p))) * D4;
  }
};

struct SrcInv {
  const float4* rows;
  const int32_t* inv;
  int D4;
  __device__ __forceinline__ const float4* operator()(int64_t t) const {
    const int32_t k = inv[t];
    return k < 0 ? nullptr : rows + (int64_t)k * D4;  // inv -1: a dropped id -> zero row
  }
};

template <int VPL, int RPW, class Src>
__global__ void __launch_bounds__(256)
k_copy_rows(Src src, int64_t n, const int32_t* n_dev, float4* __restrict__ out, int D4) {
  HP_ENTRY(SP_COPY);
  const int lane = threadIdx.x & 31;
  const int64_t lim = n_dev ? min(n, (int64_t)*n_dev) : n;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * RPW; r0 < lim;
       r0 += nw * RPW) {
    float4 x[RPW][VPL];
#pragma unroll
    for (int e = 0; e < RPW; ++e) {
      const int64_t r = r0 + e;
      const float4* s = r < lim ? src(r) : nullptr;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c4 = lane + 32 * v;
        x[e][v] = (s && c4 < D4) ? s[c4] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int e = 0; e < RPW; ++e) {
      const int64_t r = r0 + e;
      if (r >= lim) break;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c4 = lane + 32 * v;
        if (c4 < D4) out[r * D4 + c4] = x[e][v];
      }
    }
  }
  HP_SPAN_END(SP_COPY);
}

template <class Src>
int launch_copy(const Src& src, int64_t n, const int32_t* n_dev, float* out, int D,
                cudaStream_t st) {
  if (n <= 0) return HP_OK;
  const int D4 = D >> 2;
  const int sms = sm_count();
  float4* o = reinterpret_cast<float4*>(out);
  if (D4 <= 32) {
    launch_k(k_copy_rows<1, 8, Src>, dim3(grid_for(n, 64, sms * 8)), dim3(256), 0, st, src, n, n_dev, o, D4);
  } else if (D4 <= 64) {
    launch_k(k_copy_rows<2, 4, Src>, dim3(grid_for(n, 32, sms * 8)), dim3(256), 0, st, src, n, n_dev, o, D4);
  } else if (D4 <= 128) {
    launch_k(k_copy_rows<4, 2, Src>, dim3(grid_for(n, 16, sms * 8)), dim3(256), 0, st, src, n, n_dev, o, D4);
  } else if (D4 <= 256) {
    launch_k(k_copy_rows<8, 1, Src>, dim3(grid_for(n, 8, sms * 8)), dim3(256), 0, st, src, n, n_dev, o, D4);
  } else {
    launch_k(k_copy_rows<16, 1, Src>, dim3(grid_for(n, 8, sms * 8)), dim3(256), 0, st, src, n, n_dev, o, D4);
  }
  HP_LAUNCHED(1, "k_copy_rows");
  return HP_OK;
}

// Work unit `it` of a plan broadcast: (rows n, destination dst, this lane's
// position). long_only: `it` is a long segment's chunk (a partial slot), read
// from its descriptor (one load, then the positions); else a plan item.
__device__ __forceinline__ void bcast_unit(const DedupPlan& pl, int it, bool long_only,
                                           int lane, int& n, int& dst, int& pos) {
  if (long_only) {
    const int4 d = pl.part_desc[it];
    n = d.y;
    dst = d.z;
    pos = lane < n ? pl.sorted_pos[d.x + lane] : 0;
  } else {
    const int4 item = pl.items[it];
    n = item.y;
    dst = item.w < 0 ? pl.longs[-item.w - 1].z : item.z;
    pos = item.x < 0 ? -item.x - 1 : (lane < n ? pl.sorted_pos[item.x + lane] : 0);
  }
}

// ---- K5 / K6 through the plan, on TMA: out[t] = row of position t's segment.
// One warp per plan item (a segment, or a 16-row chunk of a long one): lane 0
// bulk-copies the segment's row (slab row of an apply plan / return row of a
// send plan: the item's destination, or its long segment's) global -> shared
// (cp.async.bulk, mbarrier), then lane j bulk-stores it shared -> global to the
// item's j-th position (cp.async.bulk.global.shared). Each unique row is read
// once per item instead of once per position, no id -> partition -> slab-row
// chain is walked (the plan already holds the destination), and the copies
// run on the TMA units (SASS UBLKCP) instead of 2 rows per warp through
// registers. Dropped ids (destination -1) get zero rows.
__global__ void __launch_bounds__(256)
k_bcast_rows(DedupPlan pl, const float4* __restrict__ rows, float4* __restrict__ out, int D4,
             int long_only, StitchWait wt) {
  extern __shared__ __align__(128) float4 s_rows[];  // [8 warps][D4]
  __shared__ uint64_t s_bar[8];
  HP_ENTRY(SP_COPY);
  block_wait_flags(wt, 8);  // p2p stitch: every owner applied (error bit 8 on timeout)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* my = s_rows + (size_t)w * D4;
  if (lane == 0) mbar_init(&s_bar[w], 1);
  __syncwarp();
  const uint32_t bytes = (uint32_t)D4 * 16u;
  // long_only: the chunks of long segments only (their rows were left to this
  // kernel by the apply + pull); work unit = a chunk = a partial slot f, whose
  // long segment is found by binary search over the descriptors' slot bases
  const int n_items = long_only ? pl.counters[C_PARTIALS] : pl.counters[C_ITEMS];
  uint32_t parity = 0;
  bool stored = false;
  for (int it = blockIdx.x * 8 + w; it < n_items; it += gridDim.x * 8) {
    int n, dst, pos;
    bcast_unit(pl, it, long_only, lane, n, dst, pos);
    if (dst < 0) {  // dropped ids: zero rows, plain stores
      for (int j = 0; j < n; ++j) {
        const int64_t p = __shfl_sync(0xffffffffu, pos, j);
        for (int c = lane; c < D4; c += 32) out[p * D4 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      continue;
    }
    if (stored) {  // this warp's previous stores have read the shared row
      if (lane < 32) bulk_wait_read0();
      __syncwarp();
    }
    if (lane == 0) {
      mbar_expect_tx(&s_bar[w], bytes);
      bulk_g2s(my, rows + (int64_t)dst * D4, bytes, &s_bar[w]);
    }
    mbar_wait(&s_bar[w], parity);
    parity ^= 1u;
    if (lane < n) {
      bulk_s2g(out + (int64_t)pos * D4, my, bytes);
      bulk_commit();
    }
    stored = true;
  }
  bulk_wait_read0();  // shared memory stays valid until every bulk store has read it
  HP_SPAN_END(SP_COPY);
}

// Register variant of k_bcast_rows (A/B, hp_debug_set_bcast_tma(0)): the warp
// loads the segment's row into registers (VPL float4 per lane) and stores it to
// each of the item's positions; no TMA round trip through shared memory.
template <int VPL>
__global__ void __launch_bounds__(256)
k_bcast_rows_reg(DedupPlan pl, const float4* __restrict__ rows, float4* __restrict__ out, int D4,
                 int long_only) {
  HP_ENTRY(SP_COPY);
  const int lane = threadIdx.x & 31;
  const int n_items = long_only ? pl.counters[C_PARTIALS] : pl.counters[C_ITEMS];
  for (int it = (blockIdx.x * 256 + threadIdx.x) >> 5; it < n_items; it += (gridDim.x * 256) >> 5) {
    int n, dst, pos;
    bcast_unit(pl, it, long_only, lane, n, dst, pos);
    float4 x[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int c = lane + 32 * v;
      x[v] = (dst >= 0 && c < D4) ? ldg_stream(rows + (int64_t)dst * D4 + c)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int j = 0; j < n; ++j) {
      const int64_t p = __shfl_sync(0xffffffffu, pos, j);
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int c = lane + 32 * v;
        if (c < D4) out[p * D4 + c] = x[v];
      }
    }
  }
  HP_SPAN_END(SP_COPY);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_init_rows(float* w, int64_t row_lo, int64_t nrows, int D, uint64_t seed,
                            float two_scale, float scale) {
  const int64_t n = nrows * D;
  const uint64_t mix = seed * 0xD1B54A32D192ED03ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = (uint64_t)(row_lo * D) + (uint64_t)i;  // global element index
    const float u = (float)(splitmix64(g ^ mix) >> 40) * (1.0f / 16777216.0f);
    w[i] = __fsub_rn(__fmul_rn(u, two_scale), scale);
  }
}

__global__ void k_fill(float4* x, int64_t n4, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = make_float4(v, v, v, v);
}

template <typename OutT>
__device__ __forceinline__ void store4(OutT* out, int64_t i4, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* out, int64_t i4, float4 v) {
  reinterpret_cast<float4*>(out)[i4] = v;
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* out, int64_t i4, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  reinterpret_cast<uint2*>(out)[i4] = u;
}
template <>
__device__ __forceinline__ void store4<__half>(__half* out, int64_t i4, float4 v) {
  __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  reinterpret_cast<uint2*>(out)[i4] = u;
}

template <typename OutT>
__global__ void __launch_bounds__(256)
k_scale_cast(const float* __restrict__ in, OutT* __restrict__ out, int64_t n, float scale) {
  const int64_t n4 = n >> 2;
  const float4* in4 = reinterpret_cast<const float4*>(in);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v = ldg_stream(in4 + i);
    v.x = __fmul_rn(v.x, scale);
    v.y = __fmul_rn(v.y, scale);
    v.z = __fmul_rn(v.z, scale);
    v.w = __fmul_rn(v.w, scale);
    store4<OutT>(out, i, v);
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = __fmul_rn(in[i], scale);
    if constexpr (sizeof(OutT) == 4) out[i] = v;
    else if constexpr (std::is_same<OutT, __nv_bfloat16>::value) out[i] = __float2bfloat16_rn(v);
    else out[i] = __float2half_rn(v);
  }
}

// bf16 -> OutT with scale: each element widened exactly to fp32, then x scale
// (scale 1 and fp32 out: the exact widening alone).
template <typename OutT>
__global__ void __launch_bounds__(256)
k_scale_cast_bf16(const __nv_bfloat16* __restrict__ in, OutT* __restrict__ out, int64_t n,
                  float scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n >> 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const uint2 u = reinterpret_cast<const uint2*>(in)[i];
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    float4 v = make_float4(__fmul_rn(a.x, scale), __fmul_rn(a.y, scale), __fmul_rn(b.x, scale),
                           __fmul_rn(b.y, scale));
    store4<OutT>(out, i, v);
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = __fmul_rn(__bfloat162float(in[i]), scale);
    if constexpr (sizeof(OutT) == 4) out[i] = v;
    else if constexpr (std::is_same<OutT, __nv_bfloat16>::value) out[i] = __float2bfloat16_rn(v);
    else out[i] = __float2half_rn(v);
  }
}

}  // namespace

HP_SPAN_SETTER(set_spans_rows)
int g_bcast_tma = 1;  // hp_debug_set_bcast_tma

int scale_cast_bf16(const void* in, void* out, int64_t count, int32_t out_dtype, float scale,
                    cudaStream_t st) {
  if (count <= 0) return HP_OK;
  HP_REQUIRE(((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0,
             "dense buffers must be 16-byte aligned");
  const int g = grid_for((count >> 2) + 1, 256, sm_count() * 8);
  const auto* x = static_cast<const __nv_bfloat16*>(in);
  switch (out_dtype) {
    case HP_DTYPE_F32:
      k_scale_cast_bf16<float><<<g, 256, 0, st>>>(x, static_cast<float*>(out), count, scale);
      break;
    case HP_DTYPE_BF16:
      k_scale_cast_bf16<__nv_bfloat16><<<g, 256, 0, st>>>(x, static_cast<__nv_bfloat16*>(out),
                                                          count, scale);
      break;
    case HP_DTYPE_F16:
      k_scale_cast_bf16<__half><<<g, 256, 0, st>>>(x, static_cast<__half*>(out), count, scale);
      break;
    default:
      set_error("unknown out_dtype");
      return HP_EINVAL;
  }
  HP_LAUNCHED(1, "k_scale_cast_bf16");
  return HP_OK;
}

int scale_cast(const float* in, void* out, int64_t count, int32_t out_dtype, float scale,
               cudaStream_t st) {
  if (count <= 0) return HP_OK;
  HP_REQUIRE(((uintptr_t)in & 15) == 0 && ((uintptr_t)out & 15) == 0,
             "dense buffers must be 16-byte aligned");
  const int g = grid_for((count >> 2) + 1, 256, sm_count() * 8);
  switch (out_dtype) {
    case HP_DTYPE_F32:
      if (scale == 1.0f && out == in) return HP_OK;
      k_scale_cast<float><<<g, 256, 0, st>>>(in, static_cast<float*>(out), count, scale);
      break;
    case HP_DTYPE_BF16:
      k_scale_cast<__nv_bfloat16><<<g, 256, 0, st>>>(in, static_cast<__nv_bfloat16*>(out), count,
                                                     scale);
      break;
    case HP_DTYPE_F16:
      k_scale_cast<__half><<<g, 256, 0, st>>>(in, static_cast<__half*>(out), count, scale);
      break;
    default:
      set_error("unknown out_dtype");
      return HP_EINVAL;
  }
  HP_LAUNCHED(1, "k_scale_cast");
  return HP_OK;
}

// K5 / K6 from a dedup plan in ws (built for the same T, D, V, P):
// out[t] = rows[destination of position t's segment] (see k_bcast_rows).
// hp_plan_stitch over all items, or (long_only) over the long segments' chunks
// of a fused-tree plan (the rest was pulled by the apply epilogue)
int plan_stitch(const void* ws, size_t ws_bytes, int64_t T, int32_t D, int64_t V, int32_t P,
                const float* rows, float* out, cudaStream_t stream, int long_only,
                const StitchWait* wait) {
  HP_REQUIRE(D >= 4 && D % 4 == 0 && D <= 2048, "D must be a multiple of 4 in [4, 2048]");
  HP_REQUIRE(T == 0 || (rows && out), "NULL argument");
  HP_REQUIRE(((uintptr_t)rows & 15) == 0 && ((uintptr_t)out & 15) == 0, "rows / out must be 16-byte aligned");
  if (T == 0) return HP_OK;
  DedupPlan pl;
  int rc = carve_plan(&pl, const_cast<void*>(ws), ws_bytes, T, D, V, P, 1);
  if (rc) return rc;
  restore_sorted_pos(pl);
  const int D4 = D >> 2;
  cudaStream_t st = stream;
  if (!g_bcast_tma && wait == nullptr) {
    const int g = grid_for(long_only ? T / HP_CHUNK + 2 : T + T / HP_CHUNK + 1, 8, sm_count() * 8);
    const float4* r4 = reinterpret_cast<const float4*>(rows);
    float4* o4 = reinterpret_cast<float4*>(out);
    if (D4 <= 32) launch_k(k_bcast_rows_reg<1>, dim3(g), dim3(256), 0, st, pl, r4, o4, D4, long_only);
    else if (D4 <= 64) launch_k(k_bcast_rows_reg<2>, dim3(g), dim3(256), 0, st, pl, r4, o4, D4, long_only);
    else if (D4 <= 128) launch_k(k_bcast_rows_reg<4>, dim3(g), dim3(256), 0, st, pl, r4, o4, D4, long_only);
    else if (D4 <= 256) launch_k(k_bcast_rows_reg<8>, dim3(g), dim3(256), 0, st, pl, r4, o4, D4, long_only);
    else launch_k(k_bcast_rows_reg<16>, dim3(g), dim3(256), 0, st, pl, r4, o4, D4, long_only);
    HP_LAUNCHED(1, "k_bcast_rows_reg");
    return HP_OK;
  }
  const size_t smem = (size_t)8 * D4 * 16;
  static bool configured = false;
  if (!configured) {
    HP_CUDA(cudaFuncSetAttribute(k_bcast_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 8 * 512 * 16));
    configured = true;
  }
  const int64_t work = long_only ? T / HP_CHUNK + 2 : T + T / HP_CHUNK + 1;
  const StitchWait wt = wait ? *wait : StitchWait{nullptr, nullptr, nullptr, 0, 0};
  launch_k(k_bcast_rows, dim3(grid_for(work, 8, sm_count() * 8)), dim3(256), smem, st, pl,
           reinterpret_cast<const float4*>(rows), reinterpret_cast<float4*>(out), D4, long_only, wt);
  HP_LAUNCHED(1, "k_bcast_rows");
  return HP_OK;
}
}  // namespace hp

using namespace hp;

extern "C" {

int hp_gather_rows(hp_slab slab, const int64_t* ids, int64_t n, const int32_t* n_dev, float* out,
                   void* stream) {
  HP_REQUIRE(slab.D >= 4 && slab.D % 4 == 0 && slab.D <= 2048, "D must be a multiple of 4");
  HP_REQUIRE(n == 0 || (ids && out && slab.w && slab.part_base), "NULL argument");
  SrcSlab src{reinterpret_cast<const float4*>(slab.w), slab.part_base, ids, Router(slab.V, slab.P),
              slab.V, slab.D >> 2};
  return launch_copy(src, n, n_dev, out, slab.D, static_cast<cudaStream_t>(stream));
}

int hp_stitch(const float* rows, const int32_t* inv, int64_t T, int32_t D, float* out,
              void* stream) {
  HP_REQUIRE(D >= 4 && D % 4 == 0 && D <= 2048, "D must be a multiple of 4");
  HP_REQUIRE(T == 0 || (rows && inv && out), "NULL argument");
  SrcInv src{reinterpret_cast<const float4*>(rows), inv, D >> 2};
  return launch_copy(src, T, nullptr, out, D, static_cast<cudaStream_t>(stream));
}


extern "C" int hp_plan_stitch(const void* ws, size_t ws_bytes, int64_t T, int32_t D, int64_t V,
                              int32_t P, const float* rows, float* out, void* stream) {
  return plan_stitch(ws, ws_bytes, T, D, V, P, rows, out, static_cast<cudaStream_t>(stream), 0);
}

int hp_init_rows(float* w, int64_t row_lo, int64_t nrows, int32_t D, uint64_t seed, float scale,
                 void* stream) {
  if (nrows <= 0) return HP_OK;
  HP_REQUIRE(w != nullptr && D >= 1, "bad init arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_init_rows<<<grid_for(nrows * D, 256, sm_count() * 8), 256, 0, st>>>(w, row_lo, nrows, D, seed,
                                                                         2.0f * scale, scale);
  HP_LAUNCHED(1, "k_init_rows");
  return HP_OK;
}

namespace hp {
namespace {
__global__ void k_inc(int32_t* c) { *c += 1; }
}  // namespace
}  // namespace hp

int hp_step_counter_inc(int32_t* ctr, void* stream) {
  HP_REQUIRE(ctr != nullptr, "NULL counter");
  k_inc<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(ctr);
  HP_LAUNCHED(1, "k_inc");
  return HP_OK;
}

int hp_fill(float* x, int64_t n, float value, void* stream) {
  if (n <= 0) return HP_OK;
  HP_REQUIRE(x != nullptr && n % 4 == 0 && ((uintptr_t)x & 15) == 0,
             "fill needs a 16-byte aligned buffer of 4k floats");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_fill<<<grid_for(n / 4, 256, sm_count() * 8), 256, 0, st>>>(reinterpret_cast<float4*>(x), n / 4,
                                                               value);
  HP_LAUNCHED(1, "k_fill");
  return HP_OK;
}

}  // extern "C"
