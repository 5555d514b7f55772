/*
 * hp_oracle.c — C restatement of oracle/oracle.py (TEST INFRASTRUCTURE ONLY).
 *
 * Same semantics, bit for bit (checked against the numpy oracle in
 * tests/test_oracle.py): stable grouping of ids, fixed summation tree with
 * fan-in CHUNK (oracle.tree_sum), send order ascending (owner, id), owner
 * merge in source-rank order, SGD / Adagrad / Adam with one IEEE fp32 op per
 * step (compiled with -ffp-contract=off, no FMA), stitch. OpenMP parallelises
 * over unique rows, so bench.py's CPU baseline / --impl reference uses every
 * host core. Only tests/, __graft_entry__.smoke() and bench.py may load it.
 *
 * Routing semantics follow the reference: contiguous even split
 * (sparseplan/model.py:36-44, 192-204), owners (crc32(name) % n + p) % n
 * (placement.py:95-97, 185-193) — the owner table is an input here.
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CHUNK 16

typedef struct {
  int64_t id;
  int64_t pos;
} kv_t;

static int cmp_kv(const void* a, const void* b) {
  const kv_t* x = (const kv_t*)a;
  const kv_t* y = (const kv_t*)b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* out[D] = tree sum of rows[idx[0..L)] (row stride D), oracle.tree_sum. */
static void tree_sum(const float* rows, const int64_t* idx, int64_t L, int D, float* out,
                     float* scratch /* >= (L/CHUNK + 1) * D */) {
  if (L <= CHUNK) {
    for (int c = 0; c < D; ++c) out[c] = 0.0f;
    for (int64_t j = 0; j < L; ++j) {
      const float* r = rows + idx[j] * (int64_t)D;
      for (int c = 0; c < D; ++c) out[c] = out[c] + r[c];
    }
    return;
  }
  /* level 0 from the indexed rows */
  int64_t n = (L + CHUNK - 1) / CHUNK;
  for (int64_t g = 0; g < n; ++g) {
    float* acc = scratch + g * D;
    for (int c = 0; c < D; ++c) acc[c] = 0.0f;
    const int64_t e = L - g * CHUNK < CHUNK ? L - g * CHUNK : CHUNK;
    for (int64_t j = 0; j < e; ++j) {
      const float* r = rows + idx[g * CHUNK + j] * (int64_t)D;
      for (int c = 0; c < D; ++c) acc[c] = acc[c] + r[c];
    }
  }
  /* upper levels in place */
  while (n > CHUNK) {
    const int64_t ng = (n + CHUNK - 1) / CHUNK;
    for (int64_t g = 0; g < ng; ++g) {
      float* tmp = out; /* group g reads slots >= g*CHUNK, writes slot g */
      for (int c = 0; c < D; ++c) tmp[c] = 0.0f;
      const int64_t e = n - g * CHUNK < CHUNK ? n - g * CHUNK : CHUNK;
      for (int64_t j = 0; j < e; ++j) {
        const float* r = scratch + (g * CHUNK + j) * D;
        for (int c = 0; c < D; ++c) tmp[c] = tmp[c] + r[c];
      }
      memcpy(scratch + g * D, tmp, sizeof(float) * D);
    }
    n = ng;
  }
  for (int c = 0; c < D; ++c) out[c] = 0.0f;
  for (int64_t j = 0; j < n; ++j)
    for (int c = 0; c < D; ++c) out[c] = out[c] + scratch[j * D + c];
}

static int64_t part_of(int64_t r, int64_t V, int32_t P) {
  const int64_t q = V / P, e = V % P, split = e * (q + 1);
  return r < split ? r / (q + 1) : e + (r - split) / q;
}

/* Group ids stably; return U and fill uniq[U], start[U+1], order[T] (positions
 * sorted by (id, pos)). Arrays are caller-allocated with capacity T (+1). */
static int64_t group_ids(const int64_t* ids, int64_t T, int64_t V, int64_t* uniq, int64_t* start,
                         int64_t* order) {
  kv_t* kv = (kv_t*)malloc(sizeof(kv_t) * (T > 0 ? T : 1));
  int64_t nv = 0; /* out-of-range ids are dropped (oracle.valid_ids) */
  for (int64_t i = 0; i < T; ++i) {
    if (ids[i] < 0 || ids[i] >= V) continue;
    kv[nv].id = ids[i];
    kv[nv].pos = i;
    ++nv;
  }
  T = nv;
  qsort(kv, (size_t)T, sizeof(kv_t), cmp_kv);
  int64_t U = 0;
  for (int64_t i = 0; i < T; ++i) {
    order[i] = kv[i].pos;
    if (i == 0 || kv[i].id != kv[i - 1].id) {
      uniq[U] = kv[i].id;
      start[U] = i;
      ++U;
    }
  }
  start[U] = T;
  free(kv);
  return U;
}

/* Worker K1+K2 (oracle.sort_dedup_route). Outputs in send order. */
int64_t hpo_sort_dedup_route(const int64_t* ids, const float* vals, int64_t T, int D, int64_t V,
                             int32_t P, const int32_t* owner, int32_t n, int64_t* send_ids,
                             float* send_rows, int32_t* counts, int32_t* inv,
                             int32_t* dest_counts) {
  int64_t* uniq = (int64_t*)malloc(sizeof(int64_t) * (T + 1));
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (T + 2));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (T + 1));
  const int64_t U = group_ids(ids, T, V, uniq, start, order);
  for (int64_t t = 0; t < T; ++t) inv[t] = -1;
  /* send slots: stable by owner, ids ascending within an owner */
  int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * (U + 1));
  for (int r = 0; r < n; ++r) dest_counts[r] = 0;
  for (int64_t u = 0; u < U; ++u) dest_counts[owner[part_of(uniq[u], V, P)]]++;
  int64_t* off = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int r = 0; r < n; ++r) off[r + 1] = off[r] + dest_counts[r];
  for (int64_t u = 0; u < U; ++u) slot[u] = off[owner[part_of(uniq[u], V, P)]]++;
#pragma omp parallel
  {
    float* scratch = (float*)malloc(sizeof(float) * (size_t)D * (T / CHUNK + 2));
#pragma omp for schedule(dynamic, 64)
    for (int64_t u = 0; u < U; ++u) {
      const int64_t s = slot[u];
      const int64_t L = start[u + 1] - start[u];
      tree_sum(vals, order + start[u], L, D, send_rows + s * (int64_t)D, scratch);
      send_ids[s] = uniq[u];
      counts[s] = (int32_t)L;
      for (int64_t j = start[u]; j < start[u + 1]; ++j) inv[order[j]] = (int32_t)s;
    }
    free(scratch);
  }
  free(uniq);
  free(start);
  free(order);
  free(slot);
  free(off);
  return U;
}

/* One row update, element-wise, exactly oracle.apply_* (kind 0/1/2). */
static void apply_row(int kind, float* w, float* s0, float* s1, const float* g, int D, float lr,
                      float b1, float b2, float omb1, float omb2, float eps, float lr_t) {
  for (int c = 0; c < D; ++c) {
    const float gc = g[c];
    if (kind == 0) {
      w[c] = w[c] - lr * gc;
    } else if (kind == 1) {
      s0[c] = s0[c] + gc * gc;
      w[c] = w[c] - (lr * gc) / sqrtf(s0[c]);
    } else {
      s0[c] = b1 * s0[c] + omb1 * gc;
      s1[c] = b2 * s1[c] + omb2 * (gc * gc);
      w[c] = w[c] - (lr_t * s0[c]) / (sqrtf(s1[c]) + eps);
    }
  }
}

/* Owner K4 (oracle.sparse_step's merge + apply_rows): ids/rows received,
 * concatenated in source order; full tables indexed by global row. */
int64_t hpo_merge_apply(const int64_t* ids, const float* rows, int64_t R, int D, int kind,
                        float* w, float* s0, float* s1, float scale, float lr, float b1, float b2,
                        float omb1, float omb2, float eps, float lr_t) {
  int64_t* uniq = (int64_t*)malloc(sizeof(int64_t) * (R + 1));
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (R + 2));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (R + 1));
  const int64_t U = group_ids(ids, R, INT64_MAX, uniq, start, order); /* owner ids are valid */
#pragma omp parallel
  {
    float* g = (float*)malloc(sizeof(float) * D);
    float* scratch = (float*)malloc(sizeof(float) * (size_t)D * (R / CHUNK + 2));
#pragma omp for schedule(dynamic, 64)
    for (int64_t u = 0; u < U; ++u) {
      tree_sum(rows, order + start[u], start[u + 1] - start[u], D, g, scratch);
      for (int c = 0; c < D; ++c) g[c] = g[c] * scale;
      const int64_t r = uniq[u] * (int64_t)D;
      apply_row(kind, w + r, s0 ? s0 + r : 0, s1 ? s1 + r : 0, g, D, lr, b1, b2, omb1, omb2, eps,
                lr_t);
    }
    free(g);
    free(scratch);
  }
  free(uniq);
  free(start);
  free(order);
  return U;
}

/* out[t] = w[ids[t]] (pull + stitch on a full table of V rows); a zero row for
 * a dropped (out-of-range) id (oracle.pull_rows). */
void hpo_gather(const float* w, int64_t V, const int64_t* ids, int64_t T, int D, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    if (ids[t] < 0 || ids[t] >= V)
      memset(out + t * (int64_t)D, 0, sizeof(float) * D);
    else
      memcpy(out + t * (int64_t)D, w + ids[t] * (int64_t)D, sizeof(float) * D);
  }
}

/* out = sum over k of grads[k] (sequential in rank order, fp32) * scale. */
void hpo_dense_mean(const float* const* grads, int n, int64_t S, float scale, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < S; ++i) {
    float a = 0.0f;
    for (int k = 0; k < n; ++k) a = a + grads[k][i];
    out[i] = a * scale;
  }
}

int hpo_chunk(void) { return CHUNK; }

/* Thread count of the OpenMP loops (the bench's CPU arms use every host thread,
 * also under torchrun, which exports OMP_NUM_THREADS=1). Returns the count set. */
int hpo_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}
