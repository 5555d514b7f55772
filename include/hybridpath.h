/*
 * hybridpath.h — C ABI of the B200-native hybrid-communication hot path.
 *
 * The reference (`sparseplan`, /root/reference/pkg/src/sparseplan) has no FFI:
 * its boundary is the Python API re-exported in `sparseplan/__init__.py:4-55`,
 * and the hot path it only *models* lives in `simulate.py`. Each entry point
 * below replaces one modelled operation of that path (file:line cited per
 * function); the Python package `paper_1808_02621_b200` binds them with ctypes
 * behind the reference's own names.
 *
 * Conventions
 *   - Every function returns 0 on success, a negative HP_E* code on failure;
 *     hp_last_error() gives the thread-local message. No exceptions, no exit().
 *   - All device buffers are allocated and owned by the caller (PyTorch).
 *     The library never allocates in a hot call; workspace is caller-provided
 *     and sized by the matching *_ws_bytes() query.
 *   - All work is enqueued on the caller's stream (cudaStream_t passed as
 *     void*). No host synchronisation unless the name says so.
 *   - Row ids are int64 at the boundary; a table holds V < 2^31 rows of D fp32
 *     (D % 4 == 0, D <= 2048).
 */
#ifndef HYBRIDPATH_H
#define HYBRIDPATH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_OK 0
#define HP_EINVAL (-1)   /* bad argument / unsupported shape */
#define HP_ECUDA (-2)    /* CUDA runtime error */
#define HP_ENCCL (-3)    /* NCCL error */
#define HP_EWS (-4)      /* workspace too small */

#define HP_OPT_SGD 0
#define HP_OPT_ADAGRAD 1
#define HP_OPT_ADAM 2

#define HP_DTYPE_F32 0
#define HP_DTYPE_BF16 1
#define HP_DTYPE_F16 2

/* Optimizer hyper-parameters for one step. lr_t / one_minus_beta* are
 * precomputed by the host in float64 and rounded to fp32. */
typedef struct hp_optim {
  int32_t kind;           /* HP_OPT_* */
  float lr;               /* SGD / Adagrad step size */
  float beta1, beta2;     /* Adam */
  float one_minus_beta1, one_minus_beta2;
  float eps;              /* Adam epsilon */
  float lr_t;             /* Adam bias-corrected step size for this step */
  float agg_scale;        /* 1/n ('mean') or 1 ('sum') applied to the merged gradient */
  /* Optional (graph replays): when lr_t_table is non-NULL the kernels use
   * lr_t_table[min(*step_ctr, table_len - 1)] instead of lr_t; the caller
   * advances *step_ctr on the device with hp_step_counter_inc each step. */
  const float* lr_t_table;
  const int32_t* step_ctr;
  int32_t table_len;
} hp_optim;

/* Sharded table slab owned by one rank: the rows of every partition it owns,
 * concatenated in ascending partition order. part_base[p] = first slab row of
 * partition p if owned here, else -1 (device int64[P]). */
typedef struct hp_slab {
  float* w;               /* [rows, D] */
  float* s0;              /* Adagrad accumulator or Adam m (NULL for SGD) */
  float* s1;              /* Adam v (NULL otherwise) */
  const int64_t* part_base; /* device int64[P] */
  int64_t V;              /* global rows of the table */
  int32_t P;              /* partition count */
  int32_t D;              /* row width (floats) */
} hp_slab;

int hp_version(void);
const char* hp_last_error(void);
int hp_device_sm_count(void);
/* Cumulative number of kernels this library has launched in the process. */
int64_t hp_launch_count(void);
/* Instrumentation: device buffer (>= 16 x 16 int64) that the dedup kernels fill
 * with per-phase clock64 stamps; NULL (default) disables it. */
void hp_debug_set_profile(long long* dev_buf);
/* Instrumentation: per-kernel-type spans (globaltimer ns, min start / max end)
 * into dev_buf[2 * 16] (starts pre-filled with ~0, ends with 0); NULL disables. */
void hp_debug_set_spans(unsigned long long* dev_buf);
/* Tuning: CTA size (256 | 512 | 1024) of the cluster dedup path. */
void hp_debug_set_cluster_threads(int nt);
/* Instrumentation: 1 = level 0 of K4 / K1-reduce runs as the cp.async row
 * stream (k_rowstream); 0 = the register-batched k_reduce (default). */
void hp_debug_set_rowstream(int on);
/* Instrumentation: 1 = launch the chain kernels with programmatic dependent
 * launch; 0 = full stream serialization (default). */
void hp_debug_set_pdl(int on);
/* Instrumentation: cap on row-stream CTAs per SM (shared memory left for
 * concurrently running kernels); default 4. */
void hp_debug_set_rs_ctas(int n);
/* Instrumentation: p2p owner merge/apply kernel. 2 (default) = k_owner_scan
 * (ownership + contributor lists, one thread per entry) + k_owner_rows (one
 * group per merged row); 1 = k_owner_stream (cp.async row stream, D in {128,
 * 256, 512, 1024}); 0 = k_owner_apply (one group per entry). */
void hp_debug_set_owner_stream(int on);
/* Instrumentation: k_combine grid cap when its epilogue stores to peers (0 = SM count, default). */
void hp_debug_set_combine_blocks(int n);
/* Grid of the pipelined dense allreduce (HP_DAR_PIPE; 0 = one block per SM) and
 * of the SM-store scatter (HP_DAR_SM; 0 = up to one block per SM). */
void hp_debug_set_dar_blocks(int n);
/* Grid of the SM-store reduce/gather kernel (HP_DAR_SM); 0 = two blocks per SM. */
void hp_debug_set_dar_rg_blocks(int n);
/* HP_DAR_SM: buckets per step (pieces of every chunk; the phases of one bucket
 * overlap the waits of the others), 1..16, default 1. */
void hp_debug_set_dar_buckets(int n);
/* A/B: 1 = the SM-store K7 kernels keep 16 (scatter) / 8 (reduce-gather)
 * vectors in flight per thread, so fewer CTAs saturate NVLink (fp32 in/out). */
void hp_debug_set_dar_deep(int on);
/* b > 0 (default 36) = the SM-store K7 scatter moves 32 KB pieces by TMA bulk
 * copies (global -> shared -> peer slot), b one-warp CTAs per peer chunk (fp32
 * gradients); 0 = LSU stores from ~half the SMs. Measured LM1B full step at
 * N = 2: 122 us (36 CTAs), 125 (32), 150 (28), 135 with LSU stores (the sparse
 * tables keep the SMs); N = 4: 181-184 vs 181. */
void hp_debug_set_dar_tma(int n);
/* A/B: b > 0 = the SM-store K7 reduce/gather on TMA bulk copies (b CTAs of 128
 * threads; fp32 in and out); 0 (default) = LSU loads and peer stores. */
void hp_debug_set_dar_rg_tma(int n);
/* Instrumentation: grids of the peer-store kernels (push reduce, owner rows):
 * 1 (default) = one group per item, many waves; 0 = one resident wave. */
void hp_debug_set_owner_waves(int on);
/* Instrumentation: k_reduce rows in flight per thread at 2 float4 columns (2 = default, 4, 8). */
void hp_debug_set_reduce_b(int b);
/* Spin-wait budget (clock cycles) of every exchange wait before it gives up and
 * raises an error bit; <= 0 restores the default (HP_WAIT_TIMEOUT_CYCLES or ~2 s). */
void hp_debug_set_wait_timeout(long long cycles);
/* A/B: 1 = long segments' chunks first, their upper tree levels fused into
 * k_reduce (TMA-staged, last-arriver nodes); 0 (default, measured faster in the
 * step and at scale) = sorted item order and a separate k_combine. Takes effect
 * for plans built afterwards. */
void hp_debug_set_fuse_tree(int on);
/* Plans built after the call: 1 (default) = items long-chunks-first, so the
 * n = 1 apply can run its short items on a side stream; 0 = build order. */
void hp_debug_set_split_long(int on);
/* A/B: b > 0 = the long chunks' reduce (split apply) keeps 8 rows in flight per
 * group, b blocks per SM at most; 0 (default) = the generic k_reduce. Measured:
 * the kernel alone is faster (K4+K5 34.5 -> 31 us) but the LM1B step slower
 * (38 -> 50 us): the long chain then reaches its TMA broadcast while the short
 * items and the next plan's cluster sort still hold the SMs. */
void hp_debug_set_long_b8(int on);
/* A/B: >= 1 = the split apply's long roots and the pull of their rows run as
 * one work-queue kernel (k_combine_bcast; > 1: that many CTAs, 1: a third of
 * the SMs); 0 (default) = k_combine + k_bcast_rows. Measured at LM1B N = 1:
 * 148 CTAs 38.4 us per step (they hold every SM's registers, the short items
 * wait), 96 34.7-36.4, 49 40.5-41.0, 16 69.1 vs 36.1-36.4: off. */
void hp_debug_set_cbcast(int on);
/* A/B: b > 0 = the split apply's long chunks reduced on TMA (k_reduce_long_tma,
 * one CTA per chunk, up to b CTAs per SM); 0 (default) = k_reduce. Measured:
 * K4+K5 alone 34.9 -> 31.0 us, the LM1B step 36.1 -> 48-51 us (see
 * profiles/r2_n1_chain_studies.txt): off. */
void hp_debug_set_long_tma(int n);
/* A/B: 1 = k_combine capped at 64 registers per thread (8 partial rows in
 * flight instead of 16; two 512-thread CTAs per SM); 0 (default) = 1 per SM. */
void hp_debug_set_comb_lite(int on);
/* A/B: k_reduce (local epilogues) grid cap in blocks per SM (default 16: one
 * group per item, many waves; 4 = one resident wave, groups loop over items). */
void hp_debug_set_reduce_bps(int n);
/* A/B: 1 (default) = chain kernels carry their stream's priority as a launch
 * attribute (graph node priority); 0 = plain launches. */
void hp_debug_set_launch_prio(int on);
/* A/B: hp_plan_stitch through TMA bulk copies (1, default) or registers (0). */
void hp_debug_set_bcast_tma(int on);

/* ---------------------------------------------------------------- CUDA graphs
 * Instantiate a captured cudaGraph_t (e.g. torch.cuda.CUDAGraph(keep_graph=True)
 * .raw_cuda_graph()) with cudaGraphInstantiateFlagUseNodePriority, so kernel
 * nodes keep the priority of the stream they were captured from (every chain
 * kernel carries it as a launch attribute): the step's plan building is
 * dispatched ahead of the apply kernels. Launch on the caller's stream. */
int hp_graph_instantiate(void* graph, int32_t use_node_priority, void** exec_out);
int hp_graph_launch(void* exec, void* stream);
int hp_graph_destroy(void* exec);

/* ---------------------------------------------------------------- asynchronous errors
 * Device-side failures (an id outside [0, V), a row not homed here, an exchange
 * wait that timed out) raise bits in device error words; nothing on the hot path
 * synchronises to read them. hp_err_collect ORs up to 8 such words (each shifted
 * left by shifts[i]) into a pinned, device-mapped host word with one 1-thread
 * kernel on the caller's stream (graph-capturable); the caller reads the host word
 * whenever it likes (HybridRunner: at the next step) and raises.
 * Replaces: nothing in the reference (it has no data path); TF1's SparseApply*
 * rejects out-of-range indices, which is the behaviour restored here. */
int hp_err_host_alloc(int32_t n, int32_t** host_out, int32_t** dev_out);
int hp_err_host_free(int32_t* host);
int hp_err_collect(const int32_t* const* words, const int32_t* shifts, int32_t n,
                   int32_t* dev_word, void* stream);
/* Device address of a dedup plan's error word (bit 0: id outside [0, V), dropped;
 * bit 1: row not homed on this rank). */
int hp_plan_err_ptr(const void* ws, const int32_t** out);

/* ---------------------------------------------------------------- K1 + K2
 * Sort + dedup + route of one worker's IndexedSlices.
 * Replaces: local aggregation (`placement.py:155-161`, `simulate.py:202-208`)
 *           and partition routing (`model.py:36-44,192-204`,
 *           `placement.py:95-97,185-193`).
 * Outputs (device): send_ids int64[U], send_rows f32[U,D] in send order
 * (ascending (owner[p(id)], id)), counts int32[U] multiplicity,
 * inv int32[T] send slot per position, dest_counts int32[nranks],
 * n_uniq int32[1]. Capacity: U <= T.
 * Ids outside [0, V) are dropped (never clamped onto a row): no slot, inv = -1,
 * error bit 0 of the plan (hp_plan_status / hp_plan_err_ptr).
 */
size_t hp_dedup_ws_bytes(int64_t T, int32_t D, int32_t P, int32_t nranks);
int hp_sort_dedup_route(const int64_t* ids, const float* vals, int64_t T, int32_t D,
                        int64_t V, int32_t P, const int32_t* owner, int32_t nranks,
                        int64_t* send_ids, float* send_rows, int32_t* counts, int32_t* inv,
                        int32_t* dest_counts, int32_t* n_uniq,
                        void* ws, size_t ws_bytes, void* stream);

/* Index-only half of hp_sort_dedup_route (no value rows): the dedup plan is
 * left in ws for hp_reduce_local_apply. */
int hp_dedup_plan(const int64_t* ids, int64_t T, int32_t D, int64_t V, int32_t P,
                  const int32_t* owner, int32_t nranks, int64_t* send_ids, int32_t* counts,
                  int32_t* inv, int32_t* dest_counts, int32_t* n_uniq,
                  void* ws, size_t ws_bytes, void* stream);

/* Error word of the last plan built in ws (bit 0: an id was outside [0, V),
 * bit 1: a row was not homed on this rank). Synchronises the stream. */
int hp_plan_status(const void* ws, int32_t* out_err, void* stream);

/* Device step counter for hp_optim.step_ctr: ++*ctr on the stream (1 thread). */
int hp_step_counter_inc(int32_t* ctr, void* stream);

/* ---------------------------------------------------------------- K4
 * Fused merge + scatter-apply on the owner.
 * Replaces: server aggregation + update (`simulate.py:294-323,358-367`),
 *           colocated update chain (`placement.py:151-154`).
 * rows [R, D] / ids [R] are what the owner received, concatenated in source
 * rank order; equal ids are summed in that order, scaled by agg_scale and
 * applied once to the slab (touched rows only).
 */
int hp_merge_apply(const int64_t* ids, const float* rows, int64_t R, hp_slab slab,
                   hp_optim opt, void* ws, size_t ws_bytes, void* stream);

/* Single-rank fused step (n == 1: every partition local, no exchange):
 * dedup the worker's slices and apply directly to the slab.
 * Equivalent to hp_sort_dedup_route followed by hp_merge_apply, without
 * materialising the summed rows. */
int hp_local_apply(const int64_t* ids, const float* vals, int64_t T, hp_slab slab,
                   hp_optim opt, void* ws, size_t ws_bytes, void* stream);

/* hp_merge_apply split in two so a caller can time K4 alone:
 * hp_apply_plan_build dedups ids[R] into a plan (in ws) whose destinations are
 * slab rows; hp_apply_plan then reduces rows[R, D] and applies the optimizer
 * with that plan (same stream, same R / slab). */
int hp_apply_plan_build(const int64_t* ids, int64_t R, hp_slab slab, void* ws, size_t ws_bytes,
                        void* stream);
int hp_apply_plan(const float* rows, int64_t R, hp_slab slab, hp_optim opt, void* ws,
                  size_t ws_bytes, void* stream);

/* K4 + K5 fused (n == 1): hp_apply_plan, and out[t] (t < R) = the updated row of
 * position t's id (a zero row for a dropped id). The apply epilogue writes the
 * positions of every short segment (<= 16 rows of one id) from its registers,
 * so the pull re-reads no updated row and walks no routing; the long (hot)
 * segments' positions get one TMA broadcast kernel after the apply (with the
 * row stream on: hp_plan_stitch after it). side_stream (nullable): the short
 * segments' reduce + apply + pull runs there, forked from and joined back into
 * `stream`, beside the long segments' chain (their chunks -> k_combine ->
 * broadcast) on `stream`. Replaces: update + pull (`simulate.py:195-199,294-323`). */
int hp_apply_plan_pull(const float* rows, int64_t R, hp_slab slab, hp_optim opt, float* out,
                       void* ws, size_t ws_bytes, void* stream, void* side_stream);

/* ---------------------------------------------------------------- K5 / K6
 * Gather: out[i] = slab row of global id ids[i], i < n (coalesced row copy); a
 * zero row for an id outside [0, V) or not homed on this rank.
 * Replaces: PS pull (`simulate.py:195-199`).
 * n_dev (nullable) = device count bounding i (rows i >= *n_dev are skipped). */
int hp_gather_rows(hp_slab slab, const int64_t* ids, int64_t n, const int32_t* n_dev,
                   float* out, void* stream);

/* Stitch: out[t] = rows[inv[t]] (t < T); inv[t] = -1 (a dropped id) gives a zero row.
 * Replaces the partition stitch
 * (`PAPER.md:473`, `simulate.py:317-323` "stitch" term). */
int hp_stitch(const float* rows, const int32_t* inv, int64_t T, int32_t D, float* out,
              void* stream);

/* K5 / K6 from the step's dedup plan (ws, built for the same T, D, V, P):
 * out[t] = rows[d(t)], d(t) = the plan destination of position t's segment —
 * a slab row for an apply plan (rows = the slab: the pull), a send slot for a
 * send plan (rows = the returned rows: the stitch); a zero row for a dropped id.
 * Each unique row is read once per plan item and broadcast to its positions by
 * TMA bulk copies. Replaces: PS pull + stitch (`simulate.py:195-199`). */
int hp_plan_stitch(const void* ws, size_t ws_bytes, int64_t T, int32_t D, int64_t V, int32_t P,
                   const float* rows, float* out, void* stream);

/* Deterministic table init: rows [row_lo, row_lo+nrows) of a D-wide table,
 * uniform[-scale, scale) from a counter hash of (seed, row, col). */
int hp_init_rows(float* w, int64_t row_lo, int64_t nrows, int32_t D, uint64_t seed,
                 float scale, void* stream);
int hp_fill(float* x, int64_t n, float value, void* stream);

/* ---------------------------------------------------------------- K7
 * Dense gradient allreduce fused with scale + cast.
 * Replaces: ring / hierarchical AllReduce (`simulate.py:97-135,243-261`).
 * comm may be NULL when nranks == 1 (then only scale + cast run).
 * in is fp32 [count]; out is out_dtype [count] (may alias in when fp32). */
typedef struct hp_comm_s* hp_comm_t;
int hp_dense_allreduce_scale_cast(hp_comm_t comm, float* in, void* out, int64_t count,
                                  int32_t out_dtype, float scale, void* stream);
/* Same with the input dtype explicit (SURVEY §8b's in_dtype): HP_DTYPE_F32
 * (then == the call above, in place in `in` for a non-fp32 out) or
 * HP_DTYPE_BF16: widened exactly into `scratch` (fp32 [count], 16-byte
 * aligned; may be NULL when nranks == 1), reduced there, scaled, cast to out. */
int hp_dense_allreduce_scale_cast_ex(hp_comm_t comm, const void* in, int32_t in_dtype, void* out,
                                     int64_t count, int32_t out_dtype, float scale, float* scratch,
                                     void* stream);

/* ---------------------------------------------------------------- other mechanisms
 * (SURVEY §8f baselines: the same Weights under transform_ar / transform_ps.)
 * hp_allgather: AR for a sparse Weight — AllGatherv of every worker's
 *   IndexedSlices (`simulate.py:138-180`); rank r's `bytes` land at recv + r*bytes.
 *   The concatenation is then applied locally on a full replica
 *   (hp_apply_plan_build / hp_apply_plan with agg_scale).
 * hp_dense_reduce_bcast: PS for a dense Weight — summed at its owner `root`
 *   (greedy placement, `placement.py:195-198`), scale + cast there, broadcast
 *   to every rank's out. in is clobbered on the owner. */
int hp_allgather(hp_comm_t comm, const void* send, void* recv, int64_t bytes, void* stream);
int hp_dense_reduce_bcast(hp_comm_t comm, float* in, void* out, int64_t count, int32_t out_dtype,
                          float scale, int32_t root, void* stream);

/* ---------------------------------------------------------------- comm / K3
 * One communicator per process/GPU over NCCL (NVLink 5 / NVSwitch).
 * Replaces: the modelled PS pull/push messages (`simulate.py:183-240`). */
int hp_nccl_unique_id_bytes(void);
int hp_nccl_get_unique_id(void* out /* hp_nccl_unique_id_bytes() bytes */);
int hp_comm_init(hp_comm_t* out, int32_t nranks, int32_t rank, const void* unique_id);
int hp_comm_destroy(hp_comm_t comm);
int hp_comm_size(hp_comm_t comm);
/* Asynchronous NCCL error (ncclCommGetAsyncError; host-only, never synchronises):
 * *out = ncclResult_t, 0 = success. HybridRunner polls it before every step. */
int hp_comm_status(hp_comm_t comm, int32_t* out);

/* all-to-all of one int32 per peer (device counts), graph-capturable. */
int hp_alltoall_counts(hp_comm_t comm, const int32_t* send, int32_t* recv, void* stream);

/* Push: (id, row) all-to-all-v with HOST counts (rows); send buffers are in
 * send order (dest-major), receive buffers are filled in source-rank order. */
int hp_exchange_push(hp_comm_t comm, const int64_t* send_ids, const float* send_rows,
                     const int32_t* send_counts, int64_t* recv_ids, float* recv_rows,
                     const int32_t* recv_counts, int32_t D, void* stream);

/* Pull: rows back along the reverse routes (owner -> worker), HOST counts. */
int hp_exchange_pull(hp_comm_t comm, const float* owner_rows, const int32_t* owner_counts,
                     float* worker_rows, const int32_t* worker_counts, int32_t D,
                     void* stream);

/* ---------------------------------------------------------------- K3/K4/K5 over NVLink
 * Device-initiated exchange through symmetric IPC windows (one per table per
 * rank): NVLink stores into owners' inboxes + epoch flags, sort-free owner
 * merge + apply, peer reads for the pull. No host synchronisation: a full
 * multi-GPU step can be captured in a CUDA graph.
 * Replaces: PS push/pull (`simulate.py:183-240`) and server aggregation +
 * update (`simulate.py:294-323`). */
typedef struct hp_xchg_s* hp_xchg_t;
size_t hp_xchg_window_bytes(int32_t n, int32_t D, int64_t cap, int64_t rows_cap);
/* Allocates this rank's window (slab of rows_cap x D fp32 + inboxes for n
 * sources x cap rows); returns the 64-byte cudaIpc handle and the slab pointer.
 * (n, D, cap, rows_cap) must be IDENTICAL on every rank: a rank addresses its
 * peers' inboxes with its own layout, so size rows_cap for the largest slab. */
int hp_xchg_create(hp_xchg_t* out, int32_t n, int32_t me, int32_t D, int64_t cap,
                   int64_t rows_cap, void* ipc_handle_out, void** w_out);
int hp_xchg_open_peer(hp_xchg_t x, int32_t rank, const void* ipc_handle);
int hp_xchg_destroy(hp_xchg_t x);
/* Worker, fused K1+K2+K3: dedup + route ids[T]/vals[T,D] and store every summed
 * row straight into its owner's inbox (NVLink stores) with an epoch-tagged entry
 * in the owner's slot table (glob_base[p] = slab row of partition p on its
 * owner); publishes counts, offsets and the step epoch at every owner. Outputs: send_ids[U], inv[T],
 * dest_counts[n], n_uniq[1] (device). ws sized by hp_dedup_ws_bytes. */
int hp_xchg_push(hp_xchg_t x, const int64_t* ids, const float* vals, int64_t T, int64_t V,
                 int32_t P, const int32_t* owner, const int64_t* glob_base, int64_t* send_ids,
                 int32_t* inv, int32_t* dest_counts, int32_t* n_uniq, void* ws, size_t ws_bytes,
                 void* stream);
/* The two halves of hp_xchg_push (so a plan can be built ahead of its step):
 * hp_xchg_plan dedups/routes ids into a send plan in ws; hp_xchg_push_plan
 * reduces vals with that plan and pushes (same T / V / P / ws). */
int hp_xchg_plan(hp_xchg_t x, const int64_t* ids, int64_t T, int64_t V, int32_t P,
                 const int32_t* owner, const int64_t* glob_base, int64_t* send_ids, int32_t* inv,
                 int32_t* dest_counts, int32_t* n_uniq, void* ws, size_t ws_bytes, void* stream);
/* (hp_xchg_push_plan takes the destinations hp_xchg_plan resolved from its
 * glob_base; the glob_base argument here is checked for non-NULL only.)
 * side_stream (nullable): the short segments' reduce + stores run there,
 * forked from and joined back into `stream`, beside the long segments' chunks
 * -> k_combine; the publication follows the join. */
int hp_xchg_push_plan(hp_xchg_t x, const float* vals, int64_t T, int64_t V, int32_t P,
                      const int64_t* send_ids, const int32_t* dest_counts,
                      const int64_t* glob_base, void* ws, size_t ws_bytes, void* stream,
                      void* side_stream);
/* Wait (one spinning block, bounded) until every source pushed (which = 0) or
 * every owner applied (which = 1) for this rank's current epoch. */
int hp_xchg_wait(hp_xchg_t x, int32_t which, void* stream);
/* Owner, fused K4+K5: (wait for all pushes — folded into k_owner_scan's
 * prologue,) merge in source order, apply to the slab, store each updated row
 * back into its contributors' return buffers. */
int hp_xchg_merge_apply(hp_xchg_t x, hp_slab slab, hp_optim opt, int32_t wait, void* stream);
/* Worker K6: (wait for all applies,) out[t] = returned row of send slot inv[t]. */
int hp_xchg_stitch(hp_xchg_t x, const int32_t* inv, int64_t T, float* out, int32_t wait,
                   void* stream);
/* Debug: the window's signal words (320 int32) to host memory (syncs). */
int hp_xchg_debug_sig(hp_xchg_t x, int32_t* host_out, void* stream);
/* Rows received from each source in the last push -> device int32[n] (async). */
int hp_xchg_recv_counts(hp_xchg_t x, int32_t* out_dev, void* stream);
/* Error bits (4/8: a wait timed out, 16: a received id is not homed here). After a
 * push wait timed out (4) the owner merges nothing: partially written inboxes are
 * never applied. */
int hp_xchg_status(hp_xchg_t x, int32_t* out_err, void* stream);
/* Device address of the exchange's error word (for hp_err_collect). */
int hp_xchg_err_ptr(hp_xchg_t x, const int32_t** out);
/* Worker K6 through the send plan in ws (hp_xchg_plan, same T / V / P): out[t] =
 * the returned row of position t's send slot, TMA-broadcast once per unique row
 * (k_bcast_rows); wait != 0 folds the wait for every owner's "applied" into the
 * kernel's prologue (no separate k_wait on the chain). */
int hp_xchg_stitch_plan(hp_xchg_t x, const void* ws, size_t ws_bytes, int64_t T, int64_t V,
                        int32_t P, float* out, int32_t wait, void* stream);
/* Forward pull (a lookup before the step): out[t] = the CURRENT row of global id
 * ids[t], read straight from its owner's slab over NVLink (peer loads; zero row
 * for an id outside [0, V)). owner / glob_base as in hp_xchg_plan. Call it after
 * this rank's previous step completed its stitch (every owner applied) and
 * before its next push. Replaces: the PS pull of the forward pass
 * (`simulate.py:195-199`; the reference's compute phase, `simulate.py:62`). */
int hp_xchg_pull(hp_xchg_t x, const int64_t* ids, int64_t T, int64_t V, int32_t P,
                 const int32_t* owner, const int64_t* glob_base, float* out, void* stream);
/* Device address of the return rows [cap][D] (indexed by this rank's send slot). */
int hp_xchg_ret_ptr(hp_xchg_t x, float** out);
/* Single-process emulation of n ranks (parity tests on ONE GPU): instead of
 * cudaIpc handles, peers are set from the raw window addresses of the other
 * emulated ranks' exchanges in this process. Same kernels and protocol. */
int hp_xchg_window_ptr(hp_xchg_t x, void** out);
int hp_xchg_set_peer_ptr(hp_xchg_t x, int32_t rank, void* window);

/* ---------------------------------------------------------------- K7 over NVLink
 * Dense allreduce fused with scale + cast, over peer memory: every rank stores
 * its chunks into the owners' reduce slots; each owner sums its chunk in
 * source-rank order (deterministic), scales, casts and stores the result into
 * every rank's output. Replaces: ring / hierarchical AllReduce
 * (`simulate.py:97-135,243-261`); the NCCL path stays as the baseline. */
typedef struct hp_dar_s* hp_dar_t;
int hp_dar_create(hp_dar_t* out, int32_t n, int32_t me, int64_t S, int32_t out_dtype,
                  void* ipc_handle_out, void** out_ptr);
int hp_dar_open_peer(hp_dar_t d, int32_t rank, const void* ipc_handle);
int hp_dar_destroy(hp_dar_t d);
/* grad: [S] of the window's input dtype (fp32 unless hp_dar_set_in_dtype). */
int hp_dar_allreduce(hp_dar_t d, const void* grad, float scale, void* stream);
/* Input dtype of the gradients: HP_DTYPE_F32 (default) or HP_DTYPE_BF16 (SM
 * mode only: bf16 travels over NVLink, half the bytes; every contribution is
 * widened exactly to fp32 and summed in source-rank order, then scaled and
 * cast to the output dtype). */
int hp_dar_set_in_dtype(hp_dar_t d, int32_t in_dtype);
/* Transport of the two NVLink phases: HP_DAR_SM = peer stores from SM kernels
 * (the runner's default), HP_DAR_CE = cudaMemcpyAsync peer copies on the copy
 * engines (the window's initial mode), pipelined, one-shot pull. Same result
 * bit for bit. */
#define HP_DAR_SM 0
#define HP_DAR_CE 1
#define HP_DAR_PIPE 2 /* one persistent kernel; scatter and reduce-gather pipelined by 64 KB pieces */
#define HP_DAR_PULL 3 /* one-shot: copy in, publish, read every peer's copy and sum (n <= 8; n = 2 default) */
int hp_dar_set_mode(hp_dar_t d, int32_t mode);
/* Split of the reduction between ranks: rank r reduces a share of S
 * proportional to weights[n] (double, >= 0, identical on every rank; default
 * uniform). Weight 0 takes a rank out of the reduce/gather work, so its NVLink
 * egress is S instead of 2(n-1)/n S (a rank that homes a hot sparse partition).
 * HP_DAR_SM and HP_DAR_CE; HP_DAR_PIPE needs the uniform split. */
int hp_dar_set_split(hp_dar_t d, const double* weights);

/* K7 through the NVSwitch (NVLS multicast). mc_in / mc_out: multicast
 * addresses of symmetric buffers of S elements (S a multiple of 4 n; fp32 in,
 * out_dtype out), set up by the caller (e.g. torch symmetric memory); the
 * caller's gradient is in its own copy of mc_in. pads_dev: device array of the
 * n ranks' signal-pad pointers (>= 128 ints each, zeroed once); state_dev:
 * int32[2] {epoch, error bits}, zeroed once. out = cast(scale * sum_r in_r),
 * reduced in the switch (tolerance-checked, not bit-exact). */
int hp_nvls_allreduce(const float* mc_in, void* mc_out, int64_t S, int32_t n, int32_t me,
                      int32_t out_dtype, float scale, int32_t* const* pads_dev, int32_t* state_dev,
                      void* stream);
int hp_dar_status(hp_dar_t d, int32_t* out_err, void* stream);
int hp_dar_err_ptr(hp_dar_t d, const int32_t** out);
/* Single-process emulation (see hp_xchg_set_peer_ptr). */
int hp_dar_window_ptr(hp_dar_t d, void** out);
int hp_dar_set_peer_ptr(hp_dar_t d, int32_t rank, void* window);
/* Instrumentation: raw peer throughput over the dense window (mode 0/2 store,
 * 1/3 load; 2/3 with 4 x 16 B in flight per thread). */
int hp_debug_nvlink_bench(hp_dar_t d, int32_t peer, int32_t mode, int32_t blocks, void* stream);
/* Instrumentation: per-block publication cost (peer stores + fence variant). */
int hp_debug_fence_bench(hp_dar_t d, int32_t peer, int32_t mode, int32_t blocks, int32_t per_block,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HYBRIDPATH_H */
