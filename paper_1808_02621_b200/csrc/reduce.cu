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
#include "hp_reduce.cuh"

namespace hp {
namespace {

int check_slab(const hp_slab& s, int opt) {
  HP_REQUIRE(s.w != nullptr && s.part_base != nullptr, "slab.w / slab.part_base is NULL");
  HP_REQUIRE(s.D >= 4 && s.D % 4 == 0 && s.D <= 2048, "D must be a multiple of 4 in [4, 2048]");
  HP_REQUIRE(opt == HP_OPT_SGD || s.s0 != nullptr, "optimizer state s0 is NULL");
  HP_REQUIRE(opt != HP_OPT_ADAM || s.s1 != nullptr, "Adam state s1 is NULL");
  HP_REQUIRE(opt >= HP_OPT_SGD && opt <= HP_OPT_ADAM, "unknown optimizer kind");
  return HP_OK;
}

template <int OPT>
EpiApply<OPT> make_apply(const hp_slab& s, const hp_optim& o, float* out) {
  EpiApply<OPT> e{reinterpret_cast<float4*>(s.w), reinterpret_cast<float4*>(s.s0),
                  reinterpret_cast<float4*>(s.s1), o, s.D >> 2, reinterpret_cast<float4*>(out)};
  return e;
}

// Fork / join events of the split apply (hp_apply_plan_pull with a side
// stream), per device; recorded and waited on back to back, so two suffice.
cudaEvent_t split_event(int k) {
  static cudaEvent_t ev[64][2] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!ev[dev][k]) cudaEventCreateWithFlags(&ev[dev][k], cudaEventDisableTiming);
  return ev[dev][k];
}

// out (nullable): the fused pull (the plan's items in long-first order only).
int apply_plan(const DedupPlan& pl, const float* vals, const hp_slab& s, const hp_optim& o,
               cudaStream_t st, float* out = nullptr) {
  switch (o.kind) {
    case HP_OPT_SGD: return launch_reduce(pl, vals, make_apply<HP_OPT_SGD>(s, o, out), st);
    case HP_OPT_ADAGRAD: return launch_reduce(pl, vals, make_apply<HP_OPT_ADAGRAD>(s, o, out), st);
    default: return launch_reduce(pl, vals, make_apply<HP_OPT_ADAM>(s, o, out), st);
  }
}

}  // namespace

HP_SPAN_SETTER(set_spans_reduce)

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
  restore_sorted_pos(pl);
  return apply_plan(pl, rows, slab, opt, st);
}

// Error word of the last plan built in ws (bit 0: id out of range, bit 1: row
// not homed on this rank). Synchronises the stream.
// K4 + K5 fused (n = 1): reduce + apply with the plan in ws, and out[t] = the
// updated row of position t's id (zero row for a dropped id). With a fused-
// tree plan the apply epilogue writes the positions itself (long segments: the
// root's TMA bulk stores); otherwise the pull runs after it (hp_plan_stitch).
int hp_apply_plan_pull(const float* rows, int64_t R, hp_slab slab, hp_optim opt, float* out,
                       void* ws, size_t ws_bytes, void* stream, void* side_stream) {
  int rc = check_slab(slab, opt.kind);
  if (rc) return rc;
  HP_REQUIRE(R == 0 || (rows != nullptr && out != nullptr), "rows / out is NULL");
  HP_REQUIRE(((uintptr_t)out & 15) == 0, "out must be 16-byte aligned");
  DedupPlan pl;
  if ((rc = carve_plan(&pl, ws, ws_bytes, R, slab.D, slab.V, slab.P, 1))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  restore_sorted_pos(pl);
  const bool rowstream = pl.nw > 0 && rs_stages(pl.D) > 0 && !g_rowstream_off;
  // Short segments are pulled by k_reduce's epilogue, long ones by one TMA
  // broadcast after the apply. (Measured: doing the long ones in k_combine's
  // tail behind a grid barrier needs a cooperative launch, which waited for the
  // other table's concurrent kernels to drain: 43.6 -> 76 us per step.)
  if (!rowstream && side_stream != nullptr && pl.reorder && !pl.fused && R > 0) {
    // items are long-chunks-first: the short items (apply + pull from the
    // epilogue) fork onto side_stream; the long chunks -> k_combine -> their
    // broadcast stay on stream; one join. The long chain no longer waits for
    // the short items' reduce.
    cudaStream_t ss = static_cast<cudaStream_t>(side_stream);
    cudaEvent_t fork = split_event(0), join = split_event(1);
    HP_CUDA(cudaEventRecord(fork, st));
    HP_CUDA(cudaStreamWaitEvent(ss, fork, 0));
    DedupPlan ps = pl, pg = pl;
    ps.part = 2;
    pg.part = 1;
    pg.cbcast = g_cbcast;  // the long rows' pull inside the roots' kernel (k_combine_bcast)
    if ((rc = apply_plan(ps, rows, slab, opt, ss, out))) return rc;
    HP_CUDA(cudaEventRecord(join, ss));
    if ((rc = apply_plan(pg, rows, slab, opt, st, out))) return rc;
    if (!pg.cbcast &&
        (rc = plan_stitch(ws, ws_bytes, R, slab.D, slab.V, slab.P, slab.w, out, st, 1)))
      return rc;
    HP_CUDA(cudaStreamWaitEvent(st, join, 0));
    return HP_OK;
  }
  if (!rowstream) {
    if ((rc = apply_plan(pl, rows, slab, opt, st, out))) return rc;
    return plan_stitch(ws, ws_bytes, R, slab.D, slab.V, slab.P, slab.w, out, st, 1);
  }
  if ((rc = apply_plan(pl, rows, slab, opt, st))) return rc;
  return plan_stitch(ws, ws_bytes, R, slab.D, slab.V, slab.P, slab.w, out, st, 0);
}

int hp_plan_status(const void* ws, int32_t* out_err, void* stream) {
  HP_REQUIRE(ws != nullptr && out_err != nullptr, "NULL argument");
  const int32_t* counters = static_cast<const int32_t*>(ws);  // carved first
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HP_CUDA(cudaMemcpyAsync(out_err, counters + C_ERR, 4, cudaMemcpyDeviceToHost, st));
  HP_CUDA(cudaStreamSynchronize(st));
  return HP_OK;
}

}  // extern "C"
