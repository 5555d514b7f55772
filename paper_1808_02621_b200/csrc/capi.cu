// Error reporting, version and device queries for the C ABI.
#include <atomic>
#include <string>

#include "hp_common.cuh"

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
extern int g_owner_waves;
extern int g_reduce_b;
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

}  // namespace hp

extern "C" {

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
void hp_debug_set_owner_waves(int on) { hp::g_owner_waves = on ? 1 : 0; }
void hp_debug_set_reduce_b(int b) { hp::g_reduce_b = b; }

}  // extern "C"
