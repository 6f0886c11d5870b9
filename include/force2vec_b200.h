/* include/force2vec_b200.h -- the drop-in C-ABI for Force2Vec's minibatch SGD
 * step on B200 (sm_100a).  Plain C: <stdint.h> types, pointers and sizes; no
 * C++ or torch types cross this boundary.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/core/...).  Return codes mirror the reference's
 * exception taxonomy (errors.hpp:8-40, CLI mapping force2vec.cpp:23-26):
 *   F2V_OK 0, F2V_EUSAGE 1 (UsageError), F2V_EIO 2 (IoError),
 *   F2V_ERANGE 3 (FormatError/RangeError), F2V_ENUMERICAL 4 (NumericalError),
 *   F2V_ECUDA 5 (device/driver failure), F2V_EUNSUPPORTED 6 (UnsupportedError),
 *   F2V_EERROR 7 (the base class Error).
 * f2v_last_error() returns the message the reference would have thrown, e.g.
 * "non-finite gradient for vertex 7 (epoch 0, batch 3)" (trainer.cpp:149-152,
 * 229-233).
 *
 * Threading: one context per training run, not thread-safe per context; every
 * call is synchronous (work runs on the context's own CUDA stream).  There is
 * no CPU fallback: f2v_create fails with F2V_ECUDA when no sm_100 device is
 * present.
 */
#ifndef FORCE2VEC_B200_H
#define FORCE2VEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define F2V_OK 0
#define F2V_EUSAGE 1
#define F2V_EIO 2
#define F2V_ERANGE 3
#define F2V_ENUMERICAL 4
#define F2V_ECUDA 5
#define F2V_EUNSUPPORTED 6
#define F2V_EERROR 7 /* force2vec::Error itself (errors.hpp:10-12), e.g. fit_logreg's
                        "degenerate single-class input" */

/* ForceKind, force_kernels.hpp:12 (same order) */
#define F2V_SIGMOID 0
#define F2V_TDIST 1
#define F2V_FR 2
#define F2V_FA 3
#define F2V_LINLOG 4

/* negative-sample streams */
#define F2V_SAMPLER_SPLITMIX 0 /* the reference's Rng::keyed(seed,{0x33,epoch,batch}) */
#define F2V_SAMPLER_PHILOX 1   /* Philox4x32-10 keyed by seed, counter (k,batch,epoch,shard) */

/* pair-math precision of the device epochs:
 * FAST  = fp32 dot/distance/force term, fp64 accumulation (~1e-7 of the reference);
 * EXACT = fp64 everything in the reference's operation order (bitwise in practice). */
#define F2V_PRECISION_FAST 0
#define F2V_PRECISION_EXACT 1

/* ForceModel, force_kernels.hpp:17-21 */
typedef struct {
  int32_t kind;          /* F2V_SIGMOID .. F2V_LINLOG */
  float epsilon;         /* singularity clamp, default 1e-6f */
  float repulsion_cap;   /* the clamp value when has_repulsion_cap (any value, as the
                            reference's std::optional<float>: 0 zeroes repulsion) */
  int32_t has_repulsion_cap; /* 0: std::nullopt (no clamp); default 1 with 5.0f */
} f2v_force_model;

/* TrainConfig, trainer.hpp:15-30 (+ the device-side fields of SURVEY §8b) */
typedef struct {
  uint32_t dim;          /* d */
  uint32_t batch;        /* b, clamped to n as train() does (trainer.cpp:200) */
  uint32_t negatives;    /* s, shared per batch (sampling.cpp:59) */
  float lr;
  uint32_t epochs;
  f2v_force_model model;
  uint64_t seed;
  int32_t lr_decay;      /* 0 Constant, 1 LinearToZero (trainer.cpp:212-214) */
  int32_t monitor_loss;  /* 1: per-epoch loss on the pre-update snapshot */
  int32_t sampler;       /* F2V_SAMPLER_* */
  int32_t init;          /* 0: caller's Z; 1: init_embedding (trainer.cpp:62-72) */
  uint32_t first_epoch;  /* run epochs [first_epoch, first_epoch + run_epochs) of the */
  uint32_t run_epochs;   /* `epochs`-long schedule; run_epochs 0 = through the end */
  int32_t precision;     /* F2V_PRECISION_FAST (default) or F2V_PRECISION_EXACT */
  uint32_t shards;       /* vertex shards G (0/1: the reference's single stream).  G > 1 =
                            the multi-GPU semantics: shard g owns
                            a contiguous row range cut at quantiles of deg(u) + s
                            (f2v_shard_layout), shuffles it with (seed,{0x22,epoch,g}),
                            and step t = every shard's t-th batch on one snapshot.  On a
                            context attached to peers (f2v_shard_attach) G = the world
                            size and each GPU runs its own shard; otherwise one GPU runs
                            all G shards (same results). */
  uint32_t walk_length;  /* SampleMode (sampling.hpp:12-20): 0 = one-hop (CSR neighbours),
                            k > 0 = walk mode: the context of u is a k-step random walk
                            (gen_walk, sampling.cpp:27-41) drawn on the batch stream before
                            the negatives; attractive_evals = k per non-isolated vertex */
  uint32_t first_batch;  /* batch range of ONE epoch (run_epochs == 1, one-hop, one process):
                            run only steps [first_batch, first_batch + run_batches) of epoch
                            first_epoch, starting from the context's current Z as the state
                            after step first_batch - 1 (per-step parity checks at any point
                            of an epoch); run_batches 0 = the whole epoch (the default) */
  uint32_t run_batches;
} f2v_train_config;

/* TrainCounters, trainer.hpp:83-87 */
typedef struct {
  uint64_t attractive_evals;
  uint64_t repulsive_evals;
} f2v_counters;

/* where a NumericalError happened */
typedef struct {
  uint32_t epoch;
  uint64_t batch;
  uint32_t vertex;
} f2v_failure;

typedef struct f2v_ctx f2v_ctx;

/* ------------------------------------------------------------ context */
/* device = CUDA ordinal. Returns NULL on failure (see f2v_global_error()). */
f2v_ctx* f2v_create(int32_t device);
void f2v_destroy(f2v_ctx* ctx);
const char* f2v_last_error(const f2v_ctx* ctx);
const char* f2v_global_error(void);
/* kernels launched by this context since the last reset (bench evidence) */
uint64_t f2v_kernel_launches(const f2v_ctx* ctx, int32_t reset);
/* CUDA-event timing of the last f2v_train_epochs call, on the context's
 * stream: out[0] device ms of the whole call, out[1] summed ms of the
 * persistent epoch kernels, out[2] number of epoch kernels, out[3] host
 * wall ms of the call. */
int32_t f2v_last_timing(const f2v_ctx* ctx, double* out4);

/* ---------------------------------------------- graph + embedding state */
/* CsrGraph (csr_graph.hpp:24-101): row_offsets u64[n+1], col_indices u32[nnz];
 * must be canonical (sorted, unique rows) -- use f2v_csr_from_edges. */
int32_t f2v_upload_graph(f2v_ctx* ctx, uint32_t n, const uint64_t* row_offsets,
                         const uint32_t* col_indices, uint64_t nnz);
/* EmbeddingMatrix (trainer.hpp:33-57): row-major f32[n*d] */
/* CsrGraph::from_edges (csr_graph.cpp:57-97) ON THE DEVICE into the context's
 * graph: self-loops dropped (counted), reversed arcs added when symmetrize,
 * sorted, deduplicated -- the same CSR, byte for byte, as f2v_csr_from_edges
 * (F2V_ERANGE for an endpoint >= n).  Replaces f2v_upload_graph for graphs
 * whose host build is the bottleneck (C5: 2.1B arcs). */
int32_t f2v_build_graph(f2v_ctx* ctx, const uint32_t* pairs, uint64_t m, uint32_t n,
                        int32_t symmetrize, uint64_t* nnz_out, uint64_t* duplicates_dropped,
                        uint64_t* self_loops_dropped);
/* the context's CSR (e.g. built by f2v_build_graph) copied out:
 * row_offsets_out[n + 1], col_out[nnz] */
int32_t f2v_get_graph(f2v_ctx* ctx, uint64_t* row_offsets_out, uint32_t* col_out);
int32_t f2v_set_embedding(f2v_ctx* ctx, const float* z, uint32_t n, uint32_t d);
int32_t f2v_get_embedding(f2v_ctx* ctx, float* z);
/* init_embedding (trainer.cpp:62-72): U(-0.5/d, 0.5/d) keyed (seed,{0x11}) */
int32_t f2v_init_embedding(f2v_ctx* ctx, uint32_t n, uint32_t d, uint64_t seed);
/* the configs' U(lo,hi) from Rng(seed,0) (test_trainer.cpp:18-23), on device */
int32_t f2v_uniform_embedding(f2v_ctx* ctx, uint32_t n, uint32_t d, uint64_t seed, float lo,
                              float hi);

/* --------------------------------- per-step operators (the reference seam) */
/* grad_minibatch (trainer.hpp:93-96, trainer.cpp:108-165) over the one-hop
 * minibatch {ids, negatives} against the device Z.  grads_out (nullable) is a
 * host f32[b*d]; the gradient also stays staged on the device for
 * f2v_apply_update(grads = NULL).  On a non-finite gradient returns
 * F2V_ENUMERICAL with *bad_vertex = first such vertex in batch order. */
int32_t f2v_grad_minibatch(f2v_ctx* ctx, const uint32_t* ids, uint32_t b,
                           const uint32_t* negatives, uint32_t s, f2v_force_model model,
                           float* grads_out, f2v_counters* counters, uint32_t* bad_vertex);
/* apply_update (trainer.hpp:99-100): z[ids[i]] -= eta * grads[i];
 * grads NULL = the staged gradient of the last f2v_grad_minibatch. */
int32_t f2v_apply_update(f2v_ctx* ctx, const uint32_t* ids, uint32_t b, const float* grads,
                         float eta);
/* batch_loss (trainer.hpp:103-104) on the device Z */
int32_t f2v_batch_loss(f2v_ctx* ctx, const uint32_t* ids, uint32_t b, const uint32_t* negatives,
                       uint32_t s, f2v_force_model model, double* loss_out);
/* fused grad (+loss) + apply of one batch; Z untouched when F2V_ENUMERICAL */
int32_t f2v_step(f2v_ctx* ctx, const uint32_t* ids, uint32_t b, const uint32_t* negatives,
                 uint32_t s, f2v_force_model model, float eta, double* loss_out,
                 f2v_counters* counters, uint32_t* bad_vertex);

/* ------------------------------------------------- device-resident epochs */
/* The train() epoch loop (trainer.cpp:211-249) on device: per epoch the
 * Fisher-Yates partition_epoch (sampling.cpp:7-19), the negatives, every
 * batch's grad_minibatch + batch_loss + apply_update in one persistent
 * dataflow kernel.  epoch_loss_out (nullable) gets one double per epoch run when
 * monitor_loss.  On F2V_ENUMERICAL, Z holds the state after the last
 * complete batch and *failure says where. */
int32_t f2v_train_epochs(f2v_ctx* ctx, const f2v_train_config* cfg, double* epoch_loss_out,
                         f2v_counters* counters, f2v_failure* failure);

/* train(g, cfg) (trainer.hpp:115-116) with host buffers: uploads the CSR and
 * z_inout (or initialises it, cfg->init), runs cfg->epochs epochs, copies Z
 * back.  device = CUDA ordinal. */
int32_t f2v_train(int32_t device, uint32_t n, const uint64_t* row_offsets,
                  const uint32_t* col_indices, uint64_t nnz, float* z_inout,
                  const f2v_train_config* cfg, double* epoch_loss_out, f2v_counters* counters,
                  f2v_failure* failure);

/* ------------------------------------------- host-side data formats (C++) */
/* CsrGraph::from_edges (csr_graph.cpp:57-97), parallel, byte-identical.
 * pairs = u32[2*m]; col_out capacity >= (symmetrize ? 2m : m).
 * Returns F2V_ERANGE on an out-of-range endpoint. */
int32_t f2v_csr_from_edges(const uint32_t* pairs, uint64_t m, uint32_t n, int32_t symmetrize,
                           uint64_t* row_offsets_out, uint32_t* col_out, uint64_t* nnz_out,
                           uint64_t* duplicates_dropped, uint64_t* self_loops_dropped);
/* partition_epoch (sampling.cpp:7-19) for train()'s key (seed,{0x22,epoch}) */
int32_t f2v_partition_epoch(uint32_t n, uint32_t b, uint64_t seed, uint32_t epoch,
                            uint32_t* perm_out);
/* the same permutation computed on the device (deterministic-reservation
 * Fisher-Yates, bit-identical); the one train_epochs uses every epoch */
int32_t f2v_device_partition_epoch(f2v_ctx* ctx, uint32_t n, uint32_t b, uint64_t seed,
                                   uint32_t epoch, uint32_t* perm_out);
/* the negatives of (epoch, batch[, shard]) under a sampler, host side */
int32_t f2v_negatives(int32_t sampler, uint64_t seed, uint32_t epoch, uint64_t batch,
                      uint32_t shard, uint32_t num_shards, uint32_t n, uint32_t s,
                      uint32_t* out);

/* Synthetic graph generators (BASELINE configs).  Each returns an arc list
 * (u32[2*m], caller frees with f2v_free) for f2v_csr_from_edges. */
int32_t f2v_gen_sbm(uint32_t n, int32_t blocks, double p_in, double p_out, uint64_t seed,
                    uint32_t** pairs_out, uint64_t* m_out);
int32_t f2v_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                     uint64_t seed, uint32_t** pairs_out, uint64_t* m_out);
int32_t f2v_gen_chung_lu(uint32_t n, double exponent, double min_deg, double max_deg,
                         double mean_deg, uint64_t seed, uint32_t** pairs_out, uint64_t* m_out);
int32_t f2v_gen_rgg(uint32_t n, double mean_deg, uint64_t seed, uint32_t** pairs_out,
                    uint64_t* m_out);
void f2v_free(void* p);

/* ------------------------------------- multi-GPU (vertex-partitioned shards)
 * No reference counterpart: the reference is single-process;
 * the semantics are the G-shard synchronous minibatch SGD the oracle pins
 * (orc_train with G > 1).  One process per GPU:
 *   f2v_upload_graph + f2v_set_embedding (same Z on every rank)
 *   f2v_shard_init(rank, world)      -- fixes both replica buffers
 *   f2v_shard_export(handles)        -- f2v_shard_handle_bytes() bytes
 *   (all-gather the handles across ranks, e.g. torch.distributed)
 *   f2v_shard_attach(all_handles)    -- world * f2v_shard_handle_bytes()
 *   f2v_train_epochs(cfg)            -- every rank, same cfg; each GPU runs its
 *                                       rows and stores every updated row into
 *                                       all replicas over NVLink.
 * Host-only helpers (no GPU needed): */
/* The G-shard layout of a graph: shard g owns rows
 * [lo_out[g], lo_out[g+1]) (cut at quantiles of deg(u) + negatives), its local
 * batch is batch_out[g]; combined step-major order: poff_out[t*G + g] = first
 * position of shard g's batch t, poff_out[T*G] = n.  Every output is nullable
 * (*steps_out = T alone sizes poff_out). */
int32_t f2v_shard_layout(uint32_t n, const uint64_t* row_offsets, uint32_t negatives,
                         uint32_t batch, uint32_t shards, uint32_t* lo_out, uint32_t* batch_out,
                         uint32_t* poff_out, uint32_t* steps_out);
/* partition_epoch (sampling.cpp:7-19) of one shard's n rows, keyed
 * (seed,{0x22,epoch}) when shards == 1 else (seed,{0x22,epoch,shard}) */
int32_t f2v_partition_shard(uint32_t n, uint32_t b, uint64_t seed, uint32_t epoch,
                            uint32_t shard, uint32_t shards, uint32_t* perm_out);
int32_t f2v_shard_handle_bytes(void);
int32_t f2v_shard_init(f2v_ctx* ctx, uint32_t rank, uint32_t world);
int32_t f2v_shard_export(f2v_ctx* ctx, uint8_t* handles_out);
int32_t f2v_shard_attach(f2v_ctx* ctx, const uint8_t* all_handles);
/* Per-step all-gather baseline (SURVEY §8e ladder step 1): the same G-shard
 * schedule, with each step's updated rows exchanged by ncclAllGather over
 * NVLink (NCCL loaded at run time, libnccl.so.2).  One process per GPU:
 * rank 0 calls f2v_nccl_unique_id, the caller broadcasts the 128 bytes, every
 * rank calls f2v_nccl_init, then f2v_train_epochs_allgather (cfg.shards 0 or
 * world).  Same results as f2v_train_epochs on an attached context. */
int32_t f2v_nccl_unique_id(uint8_t* unique_id_out /* 128 bytes */);
int32_t f2v_nccl_init(f2v_ctx* ctx, const uint8_t* unique_id, uint32_t rank, uint32_t world);
int32_t f2v_train_epochs_allgather(f2v_ctx* ctx, const f2v_train_config* cfg, double* loss_out,
                                   f2v_counters* counters, f2v_failure* failure);
/* rows of the device Z by id (the per-step all-gather driver, dist.py):
 * rows f32[b*d] row-major */
int32_t f2v_get_rows(f2v_ctx* ctx, const uint32_t* ids, uint32_t b, float* rows_out);
int32_t f2v_set_rows(f2v_ctx* ctx, const uint32_t* ids, uint32_t b, const float* rows);

/* ------------------------------------------------ after training
 * Embedding text I/O (embedding_io.cpp:24-100), host side.  The file format is
 * the reference's: header "n d", then n lines "vertex_id f_1 ... f_d" with the
 * shortest round-trip decimal of every float, so write + read is bitwise
 * lossless and files are byte-identical to the reference's.  Errors carry the
 * reference's messages (f2v_global_error()). */
int32_t f2v_write_embedding(const char* path, const float* z, uint32_t n, uint32_t d);
/* *z_out is allocated by the library (f2v_free) */
int32_t f2v_read_embedding(const char* path, float** z_out, uint32_t* n_out, uint32_t* d_out);
/* write_layout_tsv (embedding_io.cpp:102-124): "id\tx\ty[\tlabel]", d must be 2;
 * first_label nullable, -1 = unlabeled */
int32_t f2v_write_layout_tsv(const char* path, const float* z, uint32_t n, uint32_t d,
                             const int32_t* first_label);
/* write_layout_svg (embedding_io.cpp:126-159): an 800 x 800 scatter, one circle per
 * vertex coloured by its first label (12-colour palette); byte-identical output */
int32_t f2v_write_layout_svg(const char* path, const float* z, uint32_t n, uint32_t d,
                             const int32_t* first_label);
/* load_labels (evaluation.cpp:175-199): "vertex_id label_id" lines, '#'/'%' comments,
 * repeated vertices = multi-label.  Labels as a CSR over vertices, sorted and unique
 * per vertex: *offsets_out u64[n + 1], *ids_out (both f2v_free) */
int32_t f2v_load_labels(const char* path, uint32_t n, uint64_t** offsets_out, int32_t** ids_out,
                        int32_t* num_classes_out, int32_t* multi_label_out);

/* Evaluation (evaluation.cpp) on the device, over the context's graph and its
 * current embedding.  rng_state is the state word of the reference's Rng
 * (rng.hpp:12-53: next() adds the Weyl constant and mixes), advanced exactly as
 * the reference advances it; f2v_rng_state(seed, stream) = Rng(seed, stream). */
uint64_t f2v_rng_state(uint64_t seed, uint64_t stream);
/* kmeans (evaluation.cpp:428-438): Lloyd + k-means++ seeding, empty clusters
 * re-seeded at the farthest point, best of `restarts` by inertia.  The
 * clustering is bit-identical to the reference's (every fp64 sum in its order). */
int32_t f2v_kmeans(f2v_ctx* ctx, int32_t k, uint64_t* rng_state, int32_t restarts,
                   int32_t max_iters, int32_t* assignment_out, double* inertia_out);
/* kmeans_inertia (evaluation.cpp:440-458) */
int32_t f2v_kmeans_inertia(f2v_ctx* ctx, int32_t k, const int32_t* assignment,
                           double* inertia_out);
/* modularity (evaluation.cpp:460-483) of a clustering of the context's graph */
int32_t f2v_modularity(f2v_ctx* ctx, int32_t k, const int32_t* assignment, double* q_out);
/* best_modularity_sweep (evaluation.cpp:485-497): k in [2, min(kmax, n)] */
int32_t f2v_best_modularity_sweep(f2v_ctx* ctx, uint64_t* rng_state, int32_t kmax,
                                  int32_t* k_out, double* q_out);

/* LogRegConfig (evaluation.hpp:46-50) */
typedef struct {
  double lr;     /* 0.1 */
  int32_t iters; /* 500 */
  double l2;     /* 1e-4 */
} f2v_logreg_config;
/* fit_logreg (evaluation.cpp:93-121): features f32[rows * cols] row-major (host),
 * targets 0/1, weights_out f64[cols + 1] (bias last) */
int32_t f2v_fit_logreg(f2v_ctx* ctx, const float* features, uint64_t rows, uint32_t cols,
                       const int32_t* targets, f2v_logreg_config cfg, double* weights_out);
/* logreg_loss (evaluation.cpp:139-153) */
int32_t f2v_logreg_loss(f2v_ctx* ctx, const double* weights, const float* features,
                        uint64_t rows, uint32_t cols, const int32_t* targets, double l2,
                        double* loss_out);
/* build_link_dataset (evaluation.cpp:36-85), host: pairs as u32 triples
 * (u, v, is_edge); *train_out / *test_out allocated by the library (f2v_free) */
int32_t f2v_build_link_dataset(uint32_t n, const uint64_t* row_offsets,
                               const uint32_t* col_indices, uint64_t* rng_state,
                               uint32_t** train_out, uint64_t* ntrain_out, uint32_t** test_out,
                               uint64_t* ntest_out);
/* link_prediction_accuracy (evaluation.cpp:155-173) over the context's embedding:
 * Hadamard features, fit on train, accuracy on test; weights_out nullable */
int32_t f2v_link_prediction_accuracy(f2v_ctx* ctx, const uint32_t* train, uint64_t ntrain,
                                     const uint32_t* test, uint64_t ntest, f2v_logreg_config cfg,
                                     double* accuracy_out, double* weights_out);
/* node_classification (evaluation.cpp:217-321): labels as a CSR over vertices
 * (label_offsets u64[n + 1], label_ids sorted and unique per vertex -- what
 * load_labels produces); one-vs-rest fits run as one batch on the device */
int32_t f2v_node_classification(f2v_ctx* ctx, const uint64_t* label_offsets,
                                const int32_t* label_ids, int32_t num_classes,
                                double train_fraction, uint64_t* rng_state,
                                f2v_logreg_config cfg, double* micro_f1_out,
                                double* macro_f1_out);

#ifdef __cplusplus
}
#endif
#endif /* FORCE2VEC_B200_H */
