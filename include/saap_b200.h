/*
 * saap_b200.h — C ABI of the B200-native SAAP hot path (arXiv 2502.08246).
 *
 * This is the drop-in boundary for the reference's C++ API in
 * /root/reference/proj/core/include/saap/{partition,attention,qmodel}.hpp.
 * Every entry point below names the reference interface it replaces.  The
 * signatures use plain pointers and sizes only (no torch, no C++ types) so a
 * ctypes / cgo / JNI stub binds them directly.
 *
 * Conventions
 *  - Return value: SAAP_OK (0) or an error class.  SAAP_ERR_INVALID_ARGUMENT
 *    corresponds one-to-one with the reference throwing std::invalid_argument
 *    and carries the same message prefix (e.g. "sparse_attention: probes 17
 *    exceed bucket count 16"); saap_last_error() returns the thread-local text.
 *  - Host-pointer entry points ("drop-in" calls) are synchronous: they return
 *    after results are back in host memory, like the reference's value
 *    returns.  *_dev entry points take device pointers, are asynchronous on
 *    the context's stream and are what a serving loop / the bench uses.
 *  - Dtype contract: the reference API is f32 with fp64 math.  K/V caches are
 *    stored in bf16 (RNE-rounded at upload), attention accumulates in fp32;
 *    parity is defined on bf16-representable inputs (north star: 1e-3
 *    relative).  Assignment, IVF offsets/ids, routed bucket lists and the
 *    attention counters are bit-exact with the reference.
 *  - Head dims supported by the kernels: 32, 64, 128 (SAAP_ERR_UNSUPPORTED
 *    otherwise).  Any query-group size G >= 1.
 *  - No CPU fallback: without a usable sm_100 device every call fails with
 *    SAAP_ERR_NO_DEVICE.
 */
#ifndef SAAP_B200_H
#define SAAP_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define SAAP_API __attribute__((visibility("default")))
#else
#define SAAP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SAAP_OK 0
#define SAAP_ERR_INVALID_ARGUMENT 1 /* reference: std::invalid_argument */
#define SAAP_ERR_CUDA 2             /* CUDA runtime / launch failure */
#define SAAP_ERR_UNSUPPORTED 3      /* shape outside the kernels' envelope */
#define SAAP_ERR_NO_DEVICE 4        /* no sm_100 device: no fallback exists */
#define SAAP_ERR_IO 5               /* reference: saap::IoError; kind via saap_last_io_kind() */
#define SAAP_ERR_RUNTIME 6          /* reference: std::runtime_error (e.g. non-finite training loss) */

typedef struct saap_ctx saap_ctx;             /* device + stream + scratch */
typedef struct saap_partition saap_partition; /* saap::Partition (partition.hpp:14-23) */
typedef struct saap_qmodel saap_qmodel;       /* saap::QModel (qmodel.hpp:15-28) */
typedef struct saap_router saap_router;       /* saap::BucketRouter (attention.hpp:102-108) */
typedef struct saap_layer saap_layer;         /* n_groups ContextStores (attention.hpp:76-86) */
typedef struct saap_graph saap_graph;         /* captured decode step (CUDA graph) */
typedef struct saap_qtrainer saap_qtrainer;   /* QModel + TrainerState (qmodel.hpp:66-75) */
typedef struct saap_accum saap_accum;         /* PartialAccumulator (attention.hpp:30-39) */

/* saap::SparseAttnConfig (attention.hpp:21-25) with DenseWindow (:16-19). */
typedef struct {
    uint64_t probes;       /* l buckets per query group; 0 = window only */
    uint64_t block_size;   /* bucket scan granularity; validated, no effect */
    uint64_t sink_count;   /* must equal the store's id_offset */
    uint64_t recent_count; /* dense recent window */
} saap_sparse_cfg;

/* Counters of saap::AttnResult (attention.hpp:142-147), per query group. */
typedef struct {
    uint64_t keys_scored;
    uint64_t max_visited_bucket;
    int32_t empty_attention;
    int32_t reserved;
} saap_attn_stats;

SAAP_API const char* saap_last_error(void);
SAAP_API const char* saap_version(void);

/* ---- context ---------------------------------------------------------- */
SAAP_API int saap_ctx_create(int device, saap_ctx** out);
SAAP_API int saap_ctx_destroy(saap_ctx* ctx);
/* Launch on a caller-owned cudaStream_t (e.g. a serving loop's stream). */
SAAP_API int saap_ctx_set_stream(saap_ctx* ctx, void* cuda_stream);
SAAP_API int saap_ctx_get_stream(saap_ctx* ctx, void** cuda_stream);
SAAP_API int saap_ctx_synchronize(saap_ctx* ctx);
SAAP_API int saap_ctx_sm_count(saap_ctx* ctx, int* out);

/* ---- partitions, Q-models, routers ------------------------------------ */
/* Partition{centroids C x d f32}; replaces holding a saap::Partition. */
SAAP_API int saap_partition_create(saap_ctx* ctx, const float* centroids, uint64_t n_buckets,
                          uint64_t dim, saap_partition** out);
SAAP_API int saap_partition_destroy(saap_partition* p);

/* QModel parameters in the reference's in-memory fp64 layout
 * (qmodel.hpp:15-28): w1 d x h, b1/gamma/beta/run_mean/run_var 1 x h,
 * w2 h x C, b2 1 x C, all row-major. */
SAAP_API int saap_qmodel_create(saap_ctx* ctx, uint64_t dim, uint64_t hidden, uint64_t n_buckets,
                       const double* w1, const double* b1, const double* bn_gamma,
                       const double* bn_beta, const double* bn_run_mean,
                       const double* bn_run_var, const double* w2, const double* b2,
                       saap_qmodel** out);
SAAP_API int saap_qmodel_destroy(saap_qmodel* m);

/* CentroidRouter(partition, use_deroped)   attention.hpp:112-125 */
SAAP_API int saap_router_create_centroid(saap_ctx* ctx, const saap_partition* p, int use_deroped,
                                saap_router** out);
/* QModelRouter(model)                      attention.hpp:127-140 */
SAAP_API int saap_router_create_qmodel(saap_ctx* ctx, const saap_qmodel* m, saap_router** out);
SAAP_API int saap_router_destroy(saap_router* r);

/* BucketRouter::select(q_roped, q_deroped, l) -> l ids, score-descending,
 * ties toward the smaller id.                attention.cpp:275-315 */
SAAP_API int saap_router_select(saap_ctx* ctx, const saap_router* r, const float* q_roped,
                       const float* q_deroped, uint64_t G, uint64_t dim, uint64_t l,
                       uint32_t* out);
/* batched_bucket_select(model, q_group, l)   qmodel.cpp:485-511 (throws for
 * l outside [1, C], unlike the router which maps l=0 to {}). */
SAAP_API int saap_batched_bucket_select(saap_ctx* ctx, const saap_qmodel* m, const float* q_deroped,
                               uint64_t G, uint64_t dim, uint64_t l, uint32_t* out);

/* qmodel_forward(model, queries_deroped) eval mode (qmodel.cpp:375-377):
 * [n x C] probabilities (fp64 on the device, f32 out like Mat::to_tensor). */
SAAP_API int saap_qmodel_forward(saap_ctx* ctx, const saap_qmodel* m, const float* q_deroped,
                                 uint64_t n, uint64_t dim, float* out);
/* ---- key assignment and IVF ------------------------------------------ */
/* assign_keys(keys, partition)               partition.cpp:191-198 */
SAAP_API int saap_assign_keys(saap_ctx* ctx, const saap_partition* p, const float* keys, uint64_t n,
                     uint64_t dim, uint32_t* out);
/* build_ivf(assignment, C) -> off[C+1], idx  partition.cpp:200-223 */
SAAP_API int saap_build_ivf(saap_ctx* ctx, const uint32_t* assignment, uint64_t n, uint64_t n_buckets,
                   uint64_t* off, uint64_t* idx);
/* kmeans_train(keys, C, iters, rng, stats)  partition.cpp:52-179 (spherical
 * k-means, bit-exact).  seed_rows[C] are the caller's Rng draws in centroid
 * order: rng.sample_without_replacement(n, C) then rng.shuffle(...)
 * (partition.cpp:80-82).  objective_per_iter (iters entries), and the two
 * counters (KMeansStats, partition.hpp:52-57) may be NULL.  d <= 128. */
SAAP_API int saap_kmeans_train(saap_ctx* ctx, const float* keys, uint64_t n, uint64_t dim,
                      uint64_t n_buckets, uint64_t iters, const uint64_t* seed_rows,
                      float* centroids, double* objective_per_iter,
                      uint64_t* zero_vector_keys, uint64_t* empty_cluster_repairs);
/* ---- SAAPTNS1 artifacts (tensor_io.hpp:14-47, partition.cpp:260-296,
 * qmodel.cpp:530-589).  Host-only file I/O; loaded partitions / Q-models go
 * straight to the device.  SAAP_ERR_IO carries the IoErrorKind
 * (0 OpenFailed, 1 BadMagic, 2 BadVersion, 3 BadDtype, 4 BadShape,
 * 5 Truncated); validation failures are SAAP_ERR_INVALID_ARGUMENT with the
 * reference's message.  Readers take NULL outputs to query sizes. */
SAAP_API int saap_last_io_kind(void);
SAAP_API int saap_tensor_write(const char* path, const float* data, uint64_t rows, uint64_t dim);
SAAP_API int saap_tensor_read(const char* path, float* out, uint64_t cap, uint64_t* rows,
                              uint64_t* dim);
SAAP_API int saap_u64_write(const char* path, const uint64_t* v, uint64_t n);
SAAP_API int saap_u64_read(const char* path, uint64_t* out, uint64_t cap, uint64_t* n);
/* partition_load(path): unit-norm check, then a device partition. */
SAAP_API int saap_partition_load(saap_ctx* ctx, const char* path, saap_partition** out);
/* ivf_load(off_path, idx_path): prefix-sum check. */
SAAP_API int saap_ivf_load(const char* off_path, const char* idx_path, uint64_t* off,
                           uint64_t off_cap, uint64_t* n_off, uint64_t* idx, uint64_t idx_cap,
                           uint64_t* n_idx);
/* qmodel_save / qmodel_load: params[8] in checkpoint order (w1 [d x h], b1,
 * bn_gamma, bn_beta, bn_run_mean, bn_run_var [1 x h], w2 [h x C], b2 [1 x C]),
 * fp64 in memory, f32 on disk.  saap_qmodel_read fills dims[3] = (d, h, C)
 * and, when params (and its entries) are non-NULL, the widened parameters. */
SAAP_API int saap_qmodel_save(const char* dir, uint64_t dim, uint64_t hidden, uint64_t n_buckets,
                              const double* const* params);
SAAP_API int saap_qmodel_read(const char* dir, uint64_t* dims, double* const* params);
SAAP_API int saap_qmodel_load(saap_ctx* ctx, const char* dir, saap_qmodel** out);

/* ---- Q-model training on the device (qmodel.cpp:227-433), bit-exact
 * parameters.  params[8] in checkpoint order (see saap_qmodel_save);
 * hyper[5] = (lr, beta1, beta2, eps, bn_momentum) or NULL for the
 * TrainerState defaults; Adam moments start at zero (state.m empty). */
SAAP_API int saap_qtrainer_create(saap_ctx* ctx, uint64_t dim, uint64_t hidden, uint64_t n_buckets,
                                  const double* const* params, const double* hyper, uint64_t step,
                                  saap_qtrainer** out);
SAAP_API int saap_qtrainer_destroy(saap_qtrainer* t);
/* train_step_on_target(model, state, queries_deroped [n x dim] f32,
 * target [n x C] fp64) -> pre-step loss (kl_loss with CUDA log: within
 * 1e-12 relative of glibc's).  Throws (SAAP_ERR_RUNTIME, "train_step:
 * non-finite loss at step k") before touching the state, like the reference. */
SAAP_API int saap_qtrainer_step(saap_ctx* ctx, saap_qtrainer* t, const float* q, uint64_t n,
                                uint64_t dim, const double* target, double* loss);
SAAP_API int saap_qtrainer_read(saap_ctx* ctx, const saap_qtrainer* t, double* const* params,
                                uint64_t* step);
/* attention_target_rows(q_roped [n x dim], keys_roped [n_keys x dim],
 * assignment, C) -> [n x C] fp64 (qmodel.cpp:384-407), bit-exact. */
SAAP_API int saap_attention_target(saap_ctx* ctx, const float* q_roped, uint64_t n, uint64_t dim,
                                   const float* keys_roped, uint64_t n_keys,
                                   const uint32_t* assignment, uint64_t n_buckets, double* out);

/* ---- partial-attention accumulators (attention.hpp:27-70), fp64 on the
 * device, bit-exact with the reference.  Host f32 blocks are row-major; only
 * the absorbed rows are uploaded.  State read/write is for interop. */
SAAP_API int saap_accum_create(saap_ctx* ctx, uint64_t heads, uint64_t value_dim, saap_accum** out);
SAAP_API int saap_accum_destroy(saap_accum* a);
SAAP_API int saap_accum_read(saap_ctx* ctx, const saap_accum* a, double* out_acc, double* sumexp,
                             double* runmax);
SAAP_API int saap_accum_write(saap_ctx* ctx, saap_accum* a, const double* out_acc,
                              const double* sumexp, const double* runmax);
/* pattn_absorb(acc, q_group, keys, values, ids)          attention.cpp:85-89 */
SAAP_API int saap_pattn_absorb(saap_ctx* ctx, saap_accum* a, const float* q, uint64_t G, uint64_t dim,
                               const float* keys, const float* values, uint64_t n_keys,
                               uint64_t key_dim, uint64_t n_values, uint64_t value_dim,
                               const uint64_t* ids, uint64_t count);
/* pattn_absorb_range(acc, q_group, keys, values, begin, end)  attention.cpp:91-100 */
SAAP_API int saap_pattn_absorb_range(saap_ctx* ctx, saap_accum* a, const float* q, uint64_t G,
                                     uint64_t dim, const float* keys, const float* values,
                                     uint64_t n_keys, uint64_t key_dim, uint64_t n_values,
                                     uint64_t value_dim, uint64_t begin, uint64_t end);
/* merge_into(acc, part) / merge_partials(parts)           attention.cpp:102-139 */
SAAP_API int saap_merge_into(saap_ctx* ctx, saap_accum* a, const saap_accum* part);
SAAP_API int saap_merge_partials(saap_ctx* ctx, const saap_accum* const* parts, uint64_t n,
                                 saap_accum* out);
/* pattn_finalize(acc, &any_empty)                          attention.cpp:141-161 */
SAAP_API int saap_pattn_finalize(saap_ctx* ctx, const saap_accum* a, float* out, int* any_empty);
/* attention_over_ids(q_group, keys, values, ids, &any_empty) attention.cpp:197-203 */
SAAP_API int saap_attention_over_ids(saap_ctx* ctx, const float* q, uint64_t G, uint64_t dim,
                                     const float* keys, const float* values, uint64_t n_keys,
                                     uint64_t key_dim, uint64_t n_values, uint64_t value_dim,
                                     const uint64_t* ids, uint64_t count, float* out,
                                     int* any_empty);

/* rope_remove_block(keys, positions, {dim, base})  rope.cpp:87-90 */
SAAP_API int saap_rope_remove(saap_ctx* ctx, const float* x, uint64_t rows, uint64_t dim,
                     const uint64_t* positions, double base, float* out);

/* ---- context stores (one layer = n_groups (sequence, KV head) contexts) --
 * Device layout per group: rows [0,sink) the sink keys,
 * rows [sink, T) keys with position < T packed bucket-contiguously
 * (ascending position inside a bucket), rows [T, n) the recent tail in
 * position order; T = max(sink, n - recent_hint).  K and V are bf16. */
SAAP_API int saap_layer_create(saap_ctx* ctx, uint64_t n_groups, uint64_t dim, uint64_t n_buckets,
                      const uint64_t* n_keys, uint64_t sink, uint64_t recent_hint,
                      saap_layer** out);
/* Same with a per-group row capacity n_cap[g] >= n_keys[g] (NULL: n_keys),
 * so saap_layer_append can grow the contexts in place. */
SAAP_API int saap_layer_create_cap(saap_ctx* ctx, uint64_t n_groups, uint64_t dim, uint64_t n_buckets,
                          const uint64_t* n_keys, const uint64_t* n_cap, uint64_t sink,
                          uint64_t recent_hint, saap_layer** out);
SAAP_API int saap_layer_destroy(saap_layer* L);

/* build_context_store(keys_roped, values, rope, partition, sink)
 *                                            attention.cpp:249-255
 * Host f32 inputs, concatenated over groups (group g owns rows
 * [sum n_<g, sum n_<=g)).  keys_assign are the keys the partition sees (the
 * de-roped keys); pass NULL to de-rope keys_roped on device with rope_base.
 * parts has one partition per group. */
SAAP_API int saap_layer_build(saap_ctx* ctx, saap_layer* L, const saap_partition* const* parts,
                     const float* keys_roped, const float* values, const float* keys_assign,
                     double rope_base);
/* Same from device bf16 rows (asynchronous). */
SAAP_API int saap_layer_build_dev(saap_ctx* ctx, saap_layer* L, const saap_partition* const* parts,
                         const void* keys_roped_bf16, const void* values_bf16,
                         const void* keys_assign_bf16);
/* A ContextStore assembled field by field (attention.hpp:76-86; e.g.
 * attention_test.cpp:418-432): keys/values f32 (rounded to the bf16 cache),
 * the caller's assignment [sum_g (n_g - sink)] u32 < C, concatenated per
 * group; the IVF and the packed layout are built from it on the device. */
SAAP_API int saap_layer_build_assigned(saap_ctx* ctx, saap_layer* L,
                                       const saap_partition* const* parts, const float* keys_roped,
                                       const float* values, const uint32_t* assignment);

/* Incremental decode index: append k keys to every
 * context (device bf16 rows [n_groups x k x dim] each: roped keys, values,
 * pre-RoPE assignment keys).  The new keys are assigned exactly on the device
 * and the index (off / idx) rebuilt; packed rows never move.  Every later
 * step equals build_context_store over the grown contexts (attention.cpp:
 * 249-255); graphs captured on this layer must be re-captured. */
SAAP_API int saap_layer_append(saap_ctx* ctx, saap_layer* L, const void* keys_roped_bf16,
                               const void* values_bf16, const void* keys_assign_bf16, uint64_t k);
/* Same from host f32 rows [n_groups x k x dim] each (rounded to the bf16
 * cache on the device; synchronous). */
SAAP_API int saap_layer_append_host(saap_ctx* ctx, saap_layer* L, const float* keys_roped,
                                    const float* values, const float* keys_assign, uint64_t k);

/* Assignment engine: 0 (default) = tcgen05 bf16 two-term-split GEMM with an
 * fp64 re-check of near-tie keys (device bf16 keys, d = 128); 1 = fp64
 * CUDA-core kernel only.  Both are bit-exact with assign_keys. */
SAAP_API int saap_ctx_set_assign_mode(saap_ctx* ctx, int mode);
/* After a build: whether the tensor-core path ran, and how many keys the
 * fp64 re-check re-scored. */
SAAP_API int saap_layer_assign_info(saap_ctx* ctx, const saap_layer* L, int* used_tensor_cores,
                                    uint64_t* refined_keys);

/* Device time of the last build issued while context timing was enabled:
 * assignment (incl. fp64 re-check) and packing (histogram/scan/scatter). */
SAAP_API int saap_layer_build_timing(saap_ctx* ctx, const saap_layer* L, double* assign_ms,
                                     double* pack_ms);

/* Read back ContextStore.assignment / index for group g (host). */
SAAP_API int saap_layer_read_index(saap_ctx* ctx, const saap_layer* L, uint64_t group,
                          uint32_t* assignment, uint64_t* off, uint64_t* idx);
/* Device pointers of the packed cache (bf16 rows) for advanced callers. */
SAAP_API int saap_layer_packed_rows(const saap_layer* L, void** k_dev, void** v_dev,
                           uint64_t* total_rows);

/* sparse_attention(q_roped, q_deroped, store, router, cfg) for every group
 *                                            attention.cpp:317-376
 * Host f32 queries [n_groups x G x dim]; out [n_groups x G x dim] f32;
 * stats[n_groups]; selected (nullable) [n_groups x probes] routed buckets.
 * routers: one per group. */
SAAP_API int saap_sparse_attention(saap_ctx* ctx, const saap_layer* L,
                          const saap_router* const* routers, const float* q_roped,
                          const float* q_deroped, uint64_t G, const saap_sparse_cfg* cfg,
                          float* out, saap_attn_stats* stats, uint32_t* selected);
/* Device-pointer variant (asynchronous). */
SAAP_API int saap_sparse_attention_dev(saap_ctx* ctx, const saap_layer* L,
                              const saap_router* const* routers, const float* q_roped_dev,
                              const float* q_deroped_dev, uint64_t G,
                              const saap_sparse_cfg* cfg, float* out_dev,
                              saap_attn_stats* stats_dev, uint32_t* selected_dev);
/* sparse_attention(q_roped, q_deroped, store, router, cfg) with ANY
 * BucketRouter (attention.hpp:102-108, attention.cpp:351): the caller runs
 * router.select and passes the returned ids, selected[g * l + b] (each < C;
 * l may differ from cfg->probes, a repeated id is absorbed once per
 * occurrence on the packed-window path, like the reference).  The lists are
 * ignored where the reference does not consult the router (probes == 0, or
 * the window covers the context).  Host buffers, synchronous. */
SAAP_API int saap_sparse_attention_selected(saap_ctx* ctx, const saap_layer* L,
                                            const float* q_roped, uint64_t G,
                                            const uint32_t* selected, uint64_t l,
                                            const saap_sparse_cfg* cfg, float* out,
                                            saap_attn_stats* stats);
/* Device-pointer variant (asynchronous, graph-capturable; ids not validated:
 * each must be < C). */
SAAP_API int saap_sparse_attention_selected_dev(saap_ctx* ctx, const saap_layer* L,
                                                const float* q_roped_dev, uint64_t G,
                                                const uint32_t* selected_dev, uint64_t l,
                                                const saap_sparse_cfg* cfg, float* out_dev,
                                                saap_attn_stats* stats_dev);
/* mse(approx, exact): mean squared entrywise difference, the reference's
 * sequential fp64 sum (bit-identical).  attention.cpp:385-399 */
SAAP_API int saap_mse(const float* approx, uint64_t rows_a, uint64_t dim_a, const float* exact,
                      uint64_t rows_e, uint64_t dim_e, double* out);

/* attention_mass_coverage(q_roped, store, selected, dense) for every group
 *                                            attention.cpp:427-462
 * q [n_groups x G x dim] f32, selected [n_groups x l]; out[n_groups] (key
 * recall of the routed buckets: share of the non-window softmax mass). */
SAAP_API int saap_attention_mass_coverage(saap_ctx* ctx, const saap_layer* L, const float* q_roped,
                                          uint64_t G, const uint32_t* selected, uint64_t l,
                                          uint64_t sink, uint64_t recent, double* out);

/* full_attention(q, keys, values) over each group's whole context, from the
 * layer's packed cache (permutation-invariant)     attention.cpp:163-195 */
SAAP_API int saap_layer_full_attention(saap_ctx* ctx, const saap_layer* L, const float* q,
                              uint64_t G, float* out);

/* Dense decode baseline (the in-run comparator): a position-ordered bf16
 * KV cache already on the device, borrowed (not copied).  Group g's rows
 * start at row_base[g] and span n_keys[g] rows (host arrays).  Decoding it is
 * full_attention (attention.cpp:163-195) for every group. */
typedef struct saap_kvcache saap_kvcache;
SAAP_API int saap_kvcache_create(saap_ctx* ctx, uint64_t n_groups, uint64_t dim, const void* keys_bf16,
                        const void* values_bf16, const uint64_t* row_base,
                        const uint64_t* n_keys, saap_kvcache** out);
SAAP_API int saap_kvcache_destroy(saap_kvcache* c);
SAAP_API int saap_dense_attention_dev(saap_ctx* ctx, const saap_kvcache* c, const float* q_dev,
                             uint64_t G, float* out_dev);

/* full_attention(q, keys, values) on host f32 arrays. attention.cpp:163-195 */
SAAP_API int saap_full_attention(saap_ctx* ctx, const float* q, uint64_t G, const float* keys,
                        const float* values, uint64_t n, uint64_t dim, float* out);

/* ---- multi-GPU: KV heads sharded over ranks ----------
 * One process per GPU; rank r owns KV heads [r*H/N, (r+1)*H/N) of every
 * sequence (GQA: its query heads read no other rank's cache), so the only
 * exchange of a layer step is gathering the attention outputs.  NCCL is
 * loaded at run time (libnccl.so.2).  The reference has no multi-GPU path
 * (single-threaded CPU); this replaces running one KV cache per GPU by hand
 * (PAPER.md:539). */
typedef struct saap_comm saap_comm;
/* ncclGetUniqueId: 128 opaque bytes rank 0 hands to every rank. */
SAAP_API int saap_comm_unique_id(uint8_t* id128);
/* ncclCommInitRank on the context's device (collective). */
SAAP_API int saap_comm_init(saap_ctx* ctx, int nranks, int rank, const uint8_t* id128,
                            saap_comm** out);
SAAP_API int saap_comm_destroy(saap_comm* comm);
/* symmetric = 1 when the gather buffers are NCCL symmetric windows
 * (ncclMemAlloc + ncclCommWindowRegister, NCCL >= 2.27). */
SAAP_API int saap_comm_info(const saap_comm* comm, int* nranks, int* rank, int* symmetric,
                            int* nccl_version);
/* The communicator's (registered) send buffer of >= bytes: point the decode
 * step's outputs here and the gather starts without a copy (collective when
 * it grows). */
SAAP_API int saap_comm_send_buffer(saap_comm* comm, uint64_t bytes, void** out_dev);
/* Heads owned by `rank`: head0, heads_local (invalid if H % N != 0). */
SAAP_API int saap_shard_heads(uint64_t kv_heads, int nranks, int rank, uint64_t* head0,
                              uint64_t* heads_local);
/* All-gather of the per-rank outputs [batch][heads_local][G][d] f32 (device)
 * into [batch][nranks * heads_local][G][d] on every rank (ncclAllGather +
 * one permute kernel, on the context's stream; collective, graph-capturable
 * once the buffers exist). */
SAAP_API int saap_allgather_heads(saap_ctx* ctx, saap_comm* comm, const float* out_local_dev,
                                  uint64_t batch, uint64_t heads_local, uint64_t G, uint64_t dim,
                                  float* out_full_dev);

/* Fused output exchange over peer memory (no collective call): the step's
 * combine kernel stores every finished slot's rows straight into each rank's
 * full output buffer [batch][kv_heads][G][d] (CUDA IPC mappings: NVLink P2P
 * stores between GPUs) and bumps each rank's arrival counter (system-scope
 * release); saap_p2p_wait orders the stream after every rank's rows landed.
 * Setup: create (allocates this rank's full buffer), exchange the 64-byte
 * handles over any channel (like the NCCL id), open, attach to the context.
 * While attached, decode steps on the context deliver this way. */
typedef struct saap_p2p saap_p2p;
SAAP_API int saap_p2p_create(saap_ctx* ctx, int nranks, int rank, uint64_t full_bytes, saap_p2p** out);
SAAP_API int saap_p2p_handle(saap_p2p* p, uint8_t* handle64);
/* all_handles: nranks x 64 bytes in rank order (this rank's own entry unused). */
SAAP_API int saap_p2p_open(saap_p2p* p, const uint8_t* all_handles);
SAAP_API int saap_p2p_buffer(saap_p2p* p, void** full_out_dev);
/* Layout of this rank's groups in the full buffer: group g = seq * heads_local
 * + local head; global head = head0 + local head.  p = NULL detaches. */
SAAP_API int saap_p2p_attach(saap_ctx* ctx, saap_p2p* p, uint64_t heads_local, uint64_t head0,
                             uint64_t kv_heads);
/* Waits (on the context stream) until `arrivals` more slot deliveries reached
 * this rank (nranks x query slots per rank for one step); graph-capturable. */
SAAP_API int saap_p2p_wait(saap_ctx* ctx, saap_p2p* p, uint64_t arrivals);
/* Copies this rank's full buffer to host memory (after the context stream). */
SAAP_API int saap_p2p_read(saap_p2p* p, void* host, uint64_t bytes);
SAAP_API int saap_p2p_destroy(saap_p2p* p);

/* ---- CUDA graphs over the asynchronous calls --------------------------- */
SAAP_API int saap_graph_begin(saap_ctx* ctx);
SAAP_API int saap_graph_end(saap_ctx* ctx, saap_graph** out);
SAAP_API int saap_graph_launch(saap_ctx* ctx, saap_graph* g);
SAAP_API int saap_graph_destroy(saap_graph* g);

/* Per-kernel device timing of decode steps issued while enabled (eager
 * launches only): CUDA events bracket the route/plan kernel and the attention
 * kernel on the context stream.  saap_ctx_timing synchronizes, returns the
 * summed milliseconds and the number of steps, and clears the record. */
SAAP_API int saap_ctx_enable_timing(saap_ctx* ctx, int on);
SAAP_API int saap_ctx_timing(saap_ctx* ctx, double* route_plan_ms, double* attention_ms,
                             uint64_t* steps);

/* Kernel launches issued by this context so far (bench "gpu_launches"). */
SAAP_API int saap_ctx_launch_count(saap_ctx* ctx, uint64_t* out);
/* Tuning and diagnostics, per context (no environment variables are read):
 *   chunk (8), chunk_dense (16)   largest decode claim (tiles), sparse / dense
 *   min_chunk (4)                 smallest guided claim at the stream's end
 *   claim_lead (3), fetch_lead (2) claim the next chunk / fetch its records
 *                                 when this many tiles of the current are left
 *   inflight (0)                  0: ring depth; else max tiles issued and unconsumed
 *   tail_per_cta (1)              (unused since guided claims)
 *   decode_poll_ns (100), combine_poll_ns (1000)   polling back-off
 *   decode_wait (0)               1: decode starts after routing (no overlap)
 *   decode_tc (0)                 1: tcgen05 decode consumers (d = 128; measured slower)
 *   cluster_route (1)             0: general routing path only
 *   assign_f32_tc (1)             0: f32 assignment keys on the fp64 kernel
 *   qm_logits (0)                 Q-model logits geometry (sweeps)
 *   host_graph (1)                0: saap_sparse_attention never replays graphs
 *   debug_skip (0)                profiling only, wrong outputs: 1 no consumer math,
 *                                 2 no K/V loads
 *   trace_step / trace_decode / trace_plan (0)     saap_debug_*_trace buffers
 * Unknown names / out-of-range values: SAAP_ERR_INVALID_ARGUMENT. */
SAAP_API int saap_ctx_set_option(saap_ctx* ctx, const char* name, int64_t value);

/* ---- diagnostics ------------------------------------------------------- */
/* out[i] = the device port of glibc exp(x[i]) used by the Q-model router
 * softmax (host arrays); lets tests pin it against the host libm. */
SAAP_API int saap_debug_exp(saap_ctx* ctx, const double* x, uint64_t n, double* out);

/* With option trace_plan set: clock64 offsets of the planner's phases for
 * context 0 of the last routed decode step (16 x u64), then per fused routing
 * CTA {start, scores exchanged, selected, end (globaltimer ns), candidates,
 * 0} (6 x 1024 x u64). */
SAAP_API int saap_debug_plan_trace(saap_ctx* ctx, uint64_t* out);

/* Debug invariant: after a decode step every per-step counter and flag is
 * back at zero.  out[8]: {tickets, dynamic tiles reserved, planner CTAs,
 * published, decode CTAs exited, nonzero run counters, nonzero done/dyn
 * counters, nonzero partial/ready flags}. */
SAAP_API int saap_debug_step_state(saap_ctx* ctx, uint64_t* out);

/* With option trace_step set: reset (reset=1) or
 * read (reset=0) the step timeline: first start / last end (globaltimer ns)
 * of {approximate routing, planner, decode, combine, last run published,
 * last slot complete, -, -} (16 x u64). */
SAAP_API int saap_debug_step_trace(saap_ctx* ctx, uint64_t* out, int reset);

/* With option trace_decode set: per attention CTA of the last decode step
 * {start, first tile, end (globaltimer ns), tiles consumed, producer cycles
 * waiting for a free stage, producer cycles total, consumer cycles waiting
 * for data, producer cycles feeding work records, producer cycles waiting for
 * a record, 0 x 7} (16 x u64 each). */
SAAP_API int saap_debug_decode_trace(saap_ctx* ctx, uint64_t* out, uint64_t n_ctas);
/* With option trace_decode set: per attention CTA of the last decode step,
 * 48 tiles x {TMA issued, data landed, consumed} (globaltimer ns). */
SAAP_API int saap_debug_decode_tiles(saap_ctx* ctx, uint64_t* out, uint64_t n_ctas);

/* ---- synthetic data (bench tooling; counter-based, reproducible) ------- */
/* Fills a device bf16 [rows x dim] buffer with clustered keys / values. */
SAAP_API int saap_synth_fill_dev(saap_ctx* ctx, void* out_bf16, uint64_t rows, uint64_t dim,
                        uint64_t seed, int kind, const float* centers_dev,
                        uint64_t n_centers, float center_scale, float noise);

/* ---- synthetic benchmark inputs (the reference's generator, host code).
 * HeadSpec synthdata.hpp:24-56 (field for field; saap_head_spec_default
 * writes the reference's defaults).  Bit-identical to the reference's
 * generate_prompt on every output word; host-only (no device needed). */
typedef struct saap_head_spec {
    uint64_t dim, n_clusters;
    double key_offset, query_offset, key_center_scale, cluster_code_scale, key_noise, stable_noise,
            sink_norm, drift_rate, query_noise, query_pull, query_boost, local_boost, target_beacon,
            ood_shift, planted_longrange_fraction;
    uint64_t n_targets, local_range, longrange_threshold, window_guard, lowfreq_pairs;
    double rope_base;
    uint64_t seed;
} saap_head_spec;
SAAP_API void saap_head_spec_default(saap_head_spec* spec);
/* generate_prompt(spec, n_keys, n_q, prompt_seed)   synthdata.cpp:169-281.
 * Key/value blocks [n_keys x dim] are written as f32, or as bf16 (RNE) when
 * out_bf16 != 0; query blocks [n_q x dim] are always f32.  Any output may be
 * NULL.  planted_target: int64[n_q] (-1 = none).  threads <= 0: all cores. */
SAAP_API int saap_generate_prompt(const saap_head_spec* spec, uint64_t n_keys, uint64_t n_q,
                                  uint64_t prompt_seed, int out_bf16, void* keys_deroped,
                                  void* keys_roped, void* values, float* q_deroped, float* q_roped,
                                  int64_t* planted_target, int threads);
/* train_head_partition(spec, n_keys, n_buckets, iters, sink)  experiments.cpp:284-295:
 * the generator's partition prompt on the host, kmeans_train on the device
 * (saap_kmeans_train, bit-exact).  centroids: f32 [n_buckets x dim]. */
SAAP_API int saap_train_head_partition(saap_ctx* ctx, const saap_head_spec* spec, uint64_t n_keys,
                                       uint64_t n_buckets, uint64_t iters, uint64_t sink_count,
                                       float* centroids, int threads);

#ifdef __cplusplus
}
#endif
#endif /* SAAP_B200_H */
