// Error reporting, version and device queries for the C ABI.
#include <atomic>
#include <string>

#include <cstring>

#include "hp_dedup.cuh"

namespace hp {

extern long long* g_prof;
void set_spans_dedup(unsigned long long*);
void set_spans_reduce(unsigned long long*);
void set_spans_rows(unsigned long long*);
void set_spans_p2p(unsigned long long*);
void set_spans_nvls(unsigned long long*);
void set_cluster_threads(int nt);
extern int g_rowstream_off;
extern int g_rs_ctas;
extern int g_owner_stream;
extern int g_combine_blocks;
extern int g_dar_blocks;
extern int g_dar_buckets;
extern int g_dar_deep;
extern int g_dar_tma;
extern int g_dar_rg_tma;
extern int g_dar_rg_blocks;
extern int g_owner_waves;
extern int g_reduce_b;
extern long long g_wait_cycles;
extern int g_fuse_tree;
extern int g_split_long;
extern int g_long_b8;
extern int g_cbcast;
extern int g_long_tma;
extern int g_comb_lite;
extern int g_reduce_bps;
extern int g_bcast_tma;
int g_launch_prio = 1;
int g_pdl = 0;  // PDL measured neutral at N=1, slower at N=2

static thread_local std::string g_err;

static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return HP_ECUDA;
}

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      return 148;
  }
  return cached;
}

// ---- asynchronous error words (HybridRunner raises one step later, no host sync)
constexpr int ERR_MAX = 8;
struct ErrSrc {
  const int32_t* w[ERR_MAX];
  int32_t shift[ERR_MAX];
  int32_t n;
};
// OR the sources' device error words (shifted) into ONE host-mapped word. The
// runner gives every stream that collects its own word, so the read-modify-
// write below has a single writer.
__global__ void k_err_collect(ErrSrc s, int32_t* host_word) {
  int v = 0;
  for (int i = 0; i < s.n; ++i)
    if (s.w[i]) v |= *reinterpret_cast<const volatile int32_t*>(s.w[i]) << s.shift[i];
  if (v) {
    volatile int32_t* h = host_word;
    *h = *h | v;
  }
}

}  // namespace hp

extern "C" {

// Pinned, device-mapped host words (zeroed) for hp_err_collect.
int hp_err_host_alloc(int32_t n, int32_t** host_out, int32_t** dev_out) {
  HP_REQUIRE(n > 0 && host_out && dev_out, "bad error-word arguments");
  void* h = nullptr;
  HP_CUDA(cudaHostAlloc(&h, sizeof(int32_t) * (size_t)n, cudaHostAllocMapped));
  memset(h, 0, sizeof(int32_t) * (size_t)n);
  void* d = nullptr;
  HP_CUDA(cudaHostGetDevicePointer(&d, h, 0));
  *host_out = static_cast<int32_t*>(h);
  *dev_out = static_cast<int32_t*>(d);
  return HP_OK;
}

int hp_err_host_free(int32_t* host) {
  if (host) HP_CUDA(cudaFreeHost(host));
  return HP_OK;
}

int hp_err_collect(const int32_t* const* words, const int32_t* shifts, int32_t n,
                   int32_t* dev_word, void* stream) {
  HP_REQUIRE(n >= 0 && n <= hp::ERR_MAX && dev_word && (n == 0 || (words && shifts)),
             "bad error-collect arguments (at most 8 words)");
  hp::ErrSrc s{};
  for (int i = 0; i < n; ++i) {
    s.w[i] = words[i];
    s.shift[i] = shifts[i];
  }
  s.n = n;
  hp::k_err_collect<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(s, dev_word);
  HP_LAUNCHED(1, "k_err_collect");
  return HP_OK;
}

int hp_plan_err_ptr(const void* ws, const int32_t** out) {
  HP_REQUIRE(ws && out, "NULL argument");
  *out = static_cast<const int32_t*>(ws) + hp::C_ERR;  // counters are carved first
  return HP_OK;
}

// ---- CUDA graphs with per-node priorities (captured by the caller, e.g.
// torch.cuda.CUDAGraph(keep_graph=True) -> raw_cuda_graph()).
int hp_graph_instantiate(void* graph, int32_t use_node_priority, void** exec_out) {
  HP_REQUIRE(graph && exec_out, "NULL argument");
  cudaGraphExec_t ex = nullptr;
  // use_node_priority: 0/1 = without/with cudaGraphInstantiateFlagUseNodePriority;
  // > 1: raw cudaGraphInstantiate* flags (A/B)
  const unsigned long long flags =
      use_node_priority > 1 ? (unsigned long long)use_node_priority
                            : (use_node_priority ? cudaGraphInstantiateFlagUseNodePriority : 0);
  HP_CUDA(cudaGraphInstantiateWithFlags(&ex, static_cast<cudaGraph_t>(graph), flags));
  *exec_out = ex;
  return HP_OK;
}

int hp_graph_launch(void* exec, void* stream) {
  HP_REQUIRE(exec, "NULL graph exec");
  HP_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), static_cast<cudaStream_t>(stream)));
  return HP_OK;
}

int hp_graph_destroy(void* exec) {
  if (exec) HP_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec)));
  return HP_OK;
}

int hp_version(void) { return 100; /* 0.1.0 */ }

const char* hp_last_error(void) { return hp::g_err.c_str(); }

int hp_device_sm_count(void) { return hp::sm_count(); }

int64_t hp_launch_count(void) { return hp::g_launches.load(std::memory_order_relaxed); }

// Instrumentation only: device buffer for per-phase clock64 stamps of the dedup kernels.
void hp_debug_set_profile(long long* dev_buf) { hp::g_prof = dev_buf; }

// Instrumentation: kernel spans [first block start, last block end] (globaltimer
// ns) accumulated with atomicMin/Max into dev_buf[2 * SpanId] (SP_N entries);
// NULL disables. The caller pre-fills starts with ~0 and ends with 0.
void hp_debug_set_spans(unsigned long long* dev_buf) {
  hp::set_spans_dedup(dev_buf);
  hp::set_spans_reduce(dev_buf);
  hp::set_spans_rows(dev_buf);
  hp::set_spans_p2p(dev_buf);
  hp::set_spans_nvls(dev_buf);
}

// Tuning only: CTA size (256 | 512 | 1024) of the cluster dedup path.
void hp_debug_set_cluster_threads(int nt) { hp::set_cluster_threads(nt); }
void hp_debug_set_rowstream(int on) { hp::g_rowstream_off = on ? 0 : 1; }
void hp_debug_set_pdl(int on) { hp::g_pdl = on ? 1 : 0; }
void hp_debug_set_rs_ctas(int n) { hp::g_rs_ctas = n < 1 ? 1 : n; }
void hp_debug_set_owner_stream(int on) { hp::g_owner_stream = on < 0 ? 0 : (on > 2 ? 2 : on); }
void hp_debug_set_combine_blocks(int n) { hp::g_combine_blocks = n < 0 ? 0 : n; }
void hp_debug_set_dar_blocks(int n) { hp::g_dar_blocks = n < 0 ? 0 : n; }
void hp_debug_set_dar_rg_blocks(int n) { hp::g_dar_rg_blocks = n < 0 ? 0 : n; }
void hp_debug_set_dar_rg_tma(int n) { hp::g_dar_rg_tma = n < 0 ? 0 : n; }
void hp_debug_set_dar_tma(int n) { hp::g_dar_tma = n < 0 ? 0 : n; }
void hp_debug_set_dar_deep(int on) { hp::g_dar_deep = on ? 1 : 0; }
void hp_debug_set_dar_buckets(int n) { hp::g_dar_buckets = n < 1 ? 1 : (n > 16 ? 16 : n); }
void hp_debug_set_owner_waves(int on) { hp::g_owner_waves = on ? 1 : 0; }
void hp_debug_set_reduce_b(int b) { hp::g_reduce_b = b; }
void hp_debug_set_wait_timeout(long long cycles) { hp::g_wait_cycles = cycles; }
void hp_debug_set_fuse_tree(int on) { hp::g_fuse_tree = on ? 1 : 0; }
void hp_debug_set_reduce_bps(int n) { hp::g_reduce_bps = n < 1 ? 1 : n; }
void hp_debug_set_comb_lite(int on) { hp::g_comb_lite = on ? 1 : 0; }
void hp_debug_set_long_tma(int n) { hp::g_long_tma = n < 0 ? 0 : n; }
void hp_debug_set_cbcast(int on) { hp::g_cbcast = on < 0 ? 0 : on; }
void hp_debug_set_long_b8(int on) { hp::g_long_b8 = on < 0 ? 0 : on; }
void hp_debug_set_split_long(int on) { hp::g_split_long = on ? 1 : 0; }
void hp_debug_set_launch_prio(int on) { hp::g_launch_prio = on ? 1 : 0; }
void hp_debug_set_bcast_tma(int on) { hp::g_bcast_tma = on ? 1 : 0; }

}  // extern "C"
