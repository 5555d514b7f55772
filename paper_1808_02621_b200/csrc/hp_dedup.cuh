// Dedup plan: the index-side result of K1+K2, shared by the reduce/apply kernels.
#pragma once

#include "hp_common.cuh"

namespace hp {

// Counter slots in DedupPlan::counters (device int32).
// counters: C_QUEUE / C_DONE / C_GEN serve k_combine_bcast's work queue (zero
// after a plan build; the kernel leaves QUEUE and DONE at zero and bumps GEN)
enum { C_UNIQ = 0, C_ITEMS = 1, C_LONG = 2, C_PARTIALS = 3, C_ERR = 4, C_QUEUE = 5, C_DONE = 6,
       C_GEN = 7, C_NCOUNTERS = 8 };

// Views into the caller's workspace (all device pointers).
struct DedupPlan {
  int64_t T;            // items
  int32_t D;            // row width (floats) the partial buffer was sized for
  int32_t P, nranks;
  int64_t V;
  int32_t key_bits;     // bits of the sort key (ceil(log2 V))
  int32_t ntiles;       // large path tiles
  uint32_t* key[2];     // ping-pong sort keys [T]
  int32_t* pos[2];      // ping-pong original positions [T]
  int32_t* sorted_pos;  // alias of the final pos buffer
  uint32_t* uniq_key;   // [T] unique ids ascending (u order)
  int32_t* seg_start;   // [T+1]
  int32_t* segidx;      // [T] segment of each sorted item
  int32_t* sigma;       // [T] send slot of segment u
  int32_t* item_off;    // [T+1] first reduce item of segment u (large-path scratch)
  int4* items;          // [T] reduce items {j0, n, dst, final}: rows sorted[j0, j0+n)
  int32_t* part_off;    // [T] partial-buffer slot of segment u (large-path scratch)
  int4* longs;          // [T/C+1] long segments {partial slot, n0 chunks, dst, L rows}
  int4* part_desc;      // [2T/C+2] per partial slot (long chunk): {first sorted row, rows, dst, long index}
  int32_t* dst;         // [T] destination row of segment u (send slot or slab row)
  int32_t* long_tmp;    // [T] large-path scratch
  int32_t* first_u;     // [P+1] first unique index of partition p
  int32_t* part_base;   // [P] send-slot base of partition p
  int32_t* zero_owner;  // [P] zeros (owner table when all partitions are local)
  int32_t* tile_hist;   // [256 * ntiles]
  int32_t* digit_tot;   // [256]
  int32_t* scan_bsum;   // [scan blocks + 1]
  int32_t* counters;    // [C_NCOUNTERS]
  float* partials;      // [(2T/C + 2) * D]
  int64_t partial_rows;
  long long* prof;      // optional per-phase clock64 stamps (HP_PROFILE_PTR), else nullptr
  // Row-stream partition (k_rowstream): warp w owns the items that start in
  // sorted rows [w*R, (w+1)*R), R = ceil(T / nw); wb_item[w] / wb_row[w] are
  // its first item and that item's first sorted row. nw == 0: not used.
  int32_t nw;
  int32_t fused;        // 1: long chunks first + fused tree in k_reduce (no k_combine)
  int32_t reorder;      // 1: items long-chunks-first ([0, C_PARTIALS) long chunks, then short)
  int32_t part;         // per launch: 0 every item, 1 long chunks only, 2 short items only
  int32_t cbcast;       // per launch (part 1, local apply with the pull): k_combine_bcast
  int32_t* long_flag;   // [T/C+2] per long segment: generation its root finished (k_combine_bcast)
  int32_t* wb_item;     // [HP_RS_MAX_WARPS + 1]
  int32_t* wb_row;      // [HP_RS_MAX_WARPS + 1]
  // fused upper levels of long segments (combine_up): one arrival counter per
  // (tree node slot, level), [partial_rows][CMB_LV], zeroed with the counters
  // at every plan build and reset by each node's last arriver
  int32_t* comb_ctr;
  // p2p send plans: per send slot u {inbox index at its owner, owner rank,
  // slab row at the owner, 0}, filled on the plan stream (k_send_info) so the
  // push epilogue's destination is one independent 16-byte load
  int4* send_info;      // [T]
};

constexpr int HP_RS_MAX_WARPS = 4096;
constexpr int CMB_LV = 7;  // tree levels above the chunks (n0 <= 16^7 chunks: T < 2^31)

// Row-stream geometry for a row width of D floats: stages per warp (0 = the
// row stream does not handle this width) and warps per plan.
int rs_stages(int32_t D);
int rs_warps(int32_t D);
// Instrumentation / A-B switches (hp_debug_set_*; defaults in dedup.cu):
extern int g_rowstream_off;   // 1: level 0 runs k_reduce, 0: k_rowstream
extern int g_rs_ctas;         // row-stream CTAs per SM cap
extern int g_owner_stream;    // p2p owner merge: 0 k_owner_apply, 1 k_owner_stream, 2 scan + rows
extern int g_combine_blocks;  // k_combine grid cap for peer-store epilogues (0: SM count)
extern int g_dar_blocks;      // HP_DAR_PIPE grid (0: one block per SM)
extern int g_dar_rg_blocks;   // HP_DAR_SM reduce/gather grid (0: 2 per SM)
extern int g_dar_tma;         // > 0: K7 scatter by TMA bulk copies, that many CTAs per peer chunk
extern int g_dar_rg_tma;      // > 0: K7 reduce/gather by TMA bulk copies, that many CTAs
extern int g_dar_deep;        // SM-store K7: 16 / 8 vectors in flight per thread (A/B)
extern int g_dar_buckets;     // HP_DAR_SM buckets per step
extern int g_owner_waves;     // peer-store kernels: many waves (1) or one resident wave (0)
extern int g_reduce_b;        // k_reduce rows in flight at VPT=2 (2, 4, 8)
extern int g_reduce_bps;      // k_reduce grid cap, blocks per SM (local epilogues; default 16)
extern int g_cbcast;          // >= 1: the split apply's long roots + their pull in one kernel (A/B)
extern int g_comb_lite;       // 1: k_combine capped at 64 registers (two CTAs per SM)
extern int g_long_tma;        // > 0: long chunks reduced on TMA (k_reduce_long_tma), g per SM
extern int g_long_b8;         // > 0: long chunks reduced with 8 rows in flight (A/B; default 0)
extern int g_split_long;      // 1 (default): long-first items; the split apply / push runs the short
                              // items on a side stream beside the long chain
extern int g_fuse_tree;       // 1: fused tree (long_chunk) when the row stream is off; 0 (default)

size_t dedup_ws_bytes(int64_t T, int32_t D, int32_t P);
int carve_plan(DedupPlan* pl, void* ws, size_t ws_bytes, int64_t T, int32_t D, int64_t V,
               int32_t P, int32_t nranks);

// Build the plan on `stream`. owner == nullptr means every partition is on rank 0.
// dst_part_base (nullable): when given, a segment's destination row is its row in
// that slab (apply plans); otherwise it is the segment's send slot (send plans).
// Optional outputs (nullable): send_ids, counts, inv, dest_counts, n_uniq.
int build_plan(DedupPlan& pl, const int64_t* ids, const int32_t* owner,
               const int64_t* dst_part_base, int64_t* send_ids, int32_t* counts, int32_t* inv,
               int32_t* dest_counts, int32_t* n_uniq, cudaStream_t stream);

// Re-point pl.sorted_pos at the buffer a previous build_plan (same T, P, V) left it in.
void restore_sorted_pos(DedupPlan& pl);

}  // namespace hp
