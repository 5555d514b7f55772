// Shared helpers for the hybrid-path kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/hybridpath.h"

#define HP_CHUNK 16           // rows per sequential group of the summation tree (oracle CHUNK)
#define HP_CL_CTAS 8          // cluster sort path: CTAs per cluster (portable maximum)
#define HP_CL_THREADS 1024    // default CTA size (256 / 512 selectable for tuning)
#define HP_CL_SLICE 2048      // items per CTA
#define HP_SMALL_MAX (HP_CL_CTAS * HP_CL_SLICE)           // 16384 items
#define HP_RADIX_BITS 8
#define HP_RADIX 256
#define HP_TILE_THREADS 512   // multi-CTA sort tile
#define HP_TILE_IPT 8
#define HP_TILE (HP_TILE_THREADS * HP_TILE_IPT)          // 4096 keys per tile
#define HP_SCAN_BLOCK 1024
#define HP_SCAN_IPT 4
#define HP_SCAN_TILE (HP_SCAN_BLOCK * HP_SCAN_IPT)

namespace hp {

void set_error(const std::string& msg);
void count_launches(int n);
int cuda_fail(cudaError_t e, const char* what);

#define HP_CUDA(call)                                        \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return ::hp::cuda_fail(_e, #call); \
  } while (0)
// Check the launch(es) just issued and add them to the library's kernel-launch
// counter (hp_launch_count(): the bench's "gpu_launches" evidence).
#define HP_LAUNCHED(n, name)      \
  do {                            \
    HP_CUDA(cudaGetLastError());  \
    ::hp::count_launches(n);      \
  } while (0)
#define HP_REQUIRE(cond, msg)          \
  do {                                 \
    if (!(cond)) {                     \
      ::hp::set_error(msg);            \
      return HP_EINVAL;                \
    }                                  \
  } while (0)

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread. s_warp needs 33 ints.
// Returns the exclusive prefix; *total receives the block sum.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = warp_incl_scan(v);
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int x = lane < NW ? s_warp[lane] : 0;
    int xi = warp_incl_scan(x);
    if (lane < NW) s_warp[lane] = xi - x;
    if (lane == NW - 1) s_warp[32] = xi;
  }
  __syncthreads();
  int r = s_warp[wid] + incl - v;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

// Row id -> partition of the contiguous even split of V rows into P parts
// (reference model.py:36-44): first e = V % P parts hold q+1 rows.
struct Router {
  int64_t q, e, split;  // split = e * (q + 1)
  __host__ __device__ Router(int64_t V, int32_t P) : q(V / P), e(V % P), split((V % P) * (V / P + 1)) {}
  __device__ __forceinline__ int part(int64_t r) const {
    if (r >= 0 && r <= 0x7fffffff) {  // every in-range row (V < 2^31): 32-bit divisions
      const uint32_t u = (uint32_t)r, sp = (uint32_t)split;
      return u < sp ? (int)(u / (uint32_t)(q + 1)) : (int)(e + (u - sp) / (uint32_t)q);
    }
    return r < split ? (int)(r / (q + 1)) : (int)(e + (r - split) / q);
  }
  __device__ __forceinline__ int64_t lo(int p) const {
    return p < e ? (int64_t)p * (q + 1) : split + (int64_t)(p - e) * q;
  }
};

// Adam's bias-corrected step size: by value, or from the device table at the
// device step counter (so a captured graph sees the right step on every replay).
__device__ __forceinline__ float adam_lr_t(const hp_optim& o) {
  if (!o.lr_t_table) return o.lr_t;
  const int s = *o.step_ctr;
  return o.lr_t_table[s < o.table_len ? (s < 0 ? 0 : s) : o.table_len - 1];
}

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}

__device__ __forceinline__ float4 ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

inline int grid_for(int64_t work, int per_block, int max_blocks) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

int sm_count();

extern int g_pdl;  // programmatic dependent launch on/off (hp_debug_set_pdl)
extern int g_launch_prio;  // stream priority as a launch attribute (hp_debug_set_launch_prio)

// Chain kernels are launched with cudaLaunchKernelEx carrying the launching
// stream's priority as a per-launch attribute: captured into a CUDA graph it
// becomes the kernel NODE's priority, which a graph instantiated with
// cudaGraphInstantiateFlagUseNodePriority (hp_graph_instantiate) schedules by.
// So the next step's plan (cluster dedup, highest-priority plan stream) is
// dispatched before the table's reduce floods the SMs, instead of waiting for
// it to drain (measured: the dedup started 16 us into the step). Plus PDL when
// hp_debug_set_pdl(1).
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0, prio = 0;
  if (g_launch_prio && cudaStreamGetPriority(st, &prio) == cudaSuccess && prio != 0) {
    at[na].id = cudaLaunchAttributePriority;
    at[na].val.priority = prio;
    ++na;
  }
  if (g_pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- kernel span profiler (instrumentation only). Each TU that uses it keeps
// its own device pointer; hp_debug_set_spans() sets all of them. A kernel
// span = [first block start, last block end] in %globaltimer ns.
enum SpanId {
  SP_DEDUP = 0, SP_REDUCE, SP_COMBINE, SP_WAIT_PUSH, SP_SCATTER, SP_APPLY, SP_WAIT_APPLIED,
  SP_COPY, SP_AR_SCATTER, SP_AR_WAIT0, SP_AR_RG, SP_AR_WAIT1, SP_PUBLISH, SP_APPLIED,
  SP_REDUCE2, SP_N = 16  // SP_REDUCE2: k_reduce over the short items only (split apply)
};
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HP_SPAN_DECL static __device__ unsigned long long* d_span = nullptr;
#define HP_SPAN_BEGIN(id) \
  if (d_span && threadIdx.x == 0) atomicMin(&d_span[2 * (id)], ::hp::globaltimer())
#define HP_SPAN_END(id)                                   \
  if (d_span) {                                           \
    __syncthreads();                                      \
    if (threadIdx.x == 0) atomicMax(&d_span[2 * (id) + 1], ::hp::globaltimer()); \
  }
// Programmatic dependent launch: chain kernels are launched with launch_k
// (stream serialization relaxed) and start with HP_ENTRY, which waits for the
// previous kernel's memory (griddepcontrol.wait; a no-op for a normal launch),
// then lets the next kernel's CTAs be scheduled while this one runs. Every
// kernel launched through launch_k must execute HP_ENTRY before touching
// global memory, so completion stays transitive along the stream.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#define HP_ENTRY(id) \
  ::hp::pdl_wait();  \
  ::hp::pdl_trigger(); \
  HP_SPAN_BEGIN(id)
#define HP_SPAN_SETTER(fn) \
  void fn(unsigned long long* p) { cudaMemcpyToSymbol(d_span, &p, sizeof(p)); }
HP_SPAN_DECL

// System-scope acquire load (flags raised by peer GPUs with st.release.sys).
__device__ __forceinline__ int ld_acquire_sys_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// A bounded wait folded into a consumer kernel's prologue: every block waits
// until flags[s] >= *epoch for s < n (error bit `err_bit` on timeout).
struct StitchWait {
  const int* flags;  // nullptr: no wait
  const int* epoch;
  int* err;
  int n;
  long long cycles;
};
__device__ __forceinline__ void block_wait_flags(const StitchWait& w, int err_bit) {
  if (w.flags == nullptr) return;
  const int e = *reinterpret_cast<const volatile int*>(w.epoch);
  for (int s = threadIdx.x; s < w.n; s += blockDim.x) {
    const long long t0 = clock64();
    while (ld_acquire_sys_i32(&w.flags[s]) < e) {
      if (clock64() - t0 > w.cycles) {
        atomicOr(w.err, err_bit);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

// K5/K6 through a dedup plan (rows.cu): out[t] = rows[plan destination of t];
// long_only: only the chunks of long segments; wait: folded flag wait.
int plan_stitch(const void* ws, size_t ws_bytes, int64_t T, int32_t D, int64_t V, int32_t P,
                const float* rows, float* out, cudaStream_t stream, int long_only,
                const StitchWait* wait = nullptr);

// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) into shared memory,
// completed on an mbarrier (transaction bytes).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HP_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HP_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared, `bytes` (multiple of 16, both 16-byte aligned), completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global, `bytes` (multiple of 16, 16-byte aligned), in this thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// this thread's bulk groups: all finished reading their shared memory source
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all but the most recent bulk group have read their shared-memory source
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
// ... and fully complete (written to global memory)
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// generic-proxy writes (this thread's, and those acquired from other SMs)
// before async-proxy (TMA) reads of global memory
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

}  // namespace hp
