// K7 through the NVSwitch (NVLS): dense gradient allreduce fused with scale +
// cast, reduced inside the switch.
//
// Every rank's gradient sits in a symmetric buffer bound to a multicast object
// (set up by torch.distributed._symmetric_memory: plumbing only). Rank r owns
// chunk r: one kernel loads each 16-byte vector of its chunk with
// multimem.ld_reduce (the switch reads the n copies and returns their fp32
// sum), scales, casts, and stores the result with multimem.st (the switch
// writes it into every rank's output). Per rank NVLink bytes: ~S in + ~S out,
// independent of n (the two-phase peer exchange moves 2 S (n-1)/n each way).
// The switch's summation order is not observable, so K7 over NVLS is checked
// against the oracle within tolerance, like NCCL's.
//
// Ordering: a one-warp barrier kernel (flags in the symmetric signal pads,
// st.release.sys / ld.acquire.sys, bounded spin) before the reduce (every
// rank's input is in place) and after it (every output written; inputs free
// for the next step).
#include <cuda_bf16.h>

#include "hp_dedup.cuh"

namespace hp {
namespace {

__device__ __forceinline__ float4 mm_ld_reduce_f32x4(const void* mc) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(mc)
               : "memory");
  return r;
}

__device__ __forceinline__ void mm_st(float* mc, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void mm_st(__nv_bfloat16* mc, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  const uint32_t ua = *reinterpret_cast<uint32_t*>(&a), ub = *reinterpret_cast<uint32_t*>(&b);
  asm volatile("multimem.st.relaxed.sys.global.v2.bf16x2 [%0], {%1,%2};" ::"l"(mc), "r"(ua),
               "r"(ub)
               : "memory");
}

__device__ __forceinline__ void st_rel_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acq_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// state: [0] epoch, [1] error bits (1: barrier 0 timed out, 2: barrier 1 timed out)
// pad layout (ints, per rank): [which * 64 + source] = epoch that source reached
__global__ void k_nvls_barrier(int* const* pads, int n, int me, int* state, int which,
                               long long timeout_cycles) {
  HP_ENTRY(which ? SP_AR_WAIT1 : SP_AR_WAIT0);
  const int e = state[0] + (which == 0 ? 1 : 0);
  __threadfence_system();
  for (int t = threadIdx.x; t < n; t += blockDim.x) st_rel_sys(pads[t] + which * 64 + me, e);
  const int* mine = pads[me] + which * 64;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const long long t0 = clock64();
    while (ld_acq_sys(mine + t) < e) {
      if (clock64() - t0 > timeout_cycles) {
        atomicOr(&state[1], 1 << which);
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  if (which == 0 && threadIdx.x == 0) state[0] = e;
  HP_SPAN_END(which ? SP_AR_WAIT1 : SP_AR_WAIT0);
}

// U vectors in flight per thread (switch reductions are long-latency: 8 by
// default); chunk = S / n elements (S padded to 4n).
template <typename OutT, int U>
__global__ void __launch_bounds__(256)
k_nvls_reduce(const float* mc_in, OutT* mc_out, int64_t chunk, int me, float scale) {
  HP_ENTRY(SP_AR_RG);
  const int64_t c4 = chunk >> 2, base4 = (int64_t)me * c4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < c4; j0 += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      if (j < c4) v[u] = mm_ld_reduce_f32x4(mc_in + (base4 + j) * 4);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * stride;
      if (j >= c4) continue;
      float4 x = v[u];
      x.x = __fmul_rn(x.x, scale);
      x.y = __fmul_rn(x.y, scale);
      x.z = __fmul_rn(x.z, scale);
      x.w = __fmul_rn(x.w, scale);
      mm_st(mc_out + (base4 + j) * 4, x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) __threadfence_system();
  HP_SPAN_END(SP_AR_RG);
}

long long nvls_wait_budget() {
  static long long v = [] {
    const char* e = getenv("HP_WAIT_TIMEOUT_CYCLES");
    return e ? atoll(e) : 4000000000LL;
  }();
  return v;
}

}  // namespace

HP_SPAN_SETTER(set_spans_nvls)

}  // namespace hp

using namespace hp;

extern "C" {

int hp_nvls_allreduce(const float* mc_in, void* mc_out, int64_t S, int32_t n, int32_t me,
                      int32_t out_dtype, float scale, int32_t* const* pads_dev, int32_t* state_dev,
                      void* stream) {
  HP_REQUIRE(mc_in && mc_out && pads_dev && state_dev, "NULL argument");
  HP_REQUIRE(n >= 1 && n <= 64 && me >= 0 && me < n, "bad rank arguments");
  HP_REQUIRE(S > 0 && S % (4 * (int64_t)n) == 0, "S must be a positive multiple of 4 * n");
  HP_REQUIRE(((uintptr_t)mc_in & 15) == 0 && ((uintptr_t)mc_out & 15) == 0,
             "multicast buffers must be 16-byte aligned");
  HP_REQUIRE(out_dtype == HP_DTYPE_F32 || out_dtype == HP_DTYPE_BF16, "out dtype f32 | bf16");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t chunk = S / n;
  launch_k(k_nvls_barrier, dim3(1), dim3(32), 0, st, pads_dev, n, me, state_dev, 0,
           nvls_wait_budget());
  const int blocks = grid_for(chunk / 32, 256, g_dar_blocks > 0 ? g_dar_blocks : sm_count() * 4);
  if (out_dtype == HP_DTYPE_F32)
    launch_k(k_nvls_reduce<float, 8>, dim3(blocks), dim3(256), 0, st, mc_in,
             static_cast<float*>(mc_out), chunk, me, scale);
  else
    launch_k(k_nvls_reduce<__nv_bfloat16, 8>, dim3(blocks), dim3(256), 0, st, mc_in,
             static_cast<__nv_bfloat16*>(mc_out), chunk, me, scale);
  launch_k(k_nvls_barrier, dim3(1), dim3(32), 0, st, pads_dev, n, me, state_dev, 1,
           nvls_wait_budget());
  HP_LAUNCHED(3, "dense nvls allreduce");
  return HP_OK;
}

}  // extern "C"
