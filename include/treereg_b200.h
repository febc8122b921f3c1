/* treereg_b200.h — C-ABI of the B200-native HGMR hot path.
 *
 * Drop-in boundary for the reference's C++ hot-path API (namespace treereg,
 * /root/reference/proj/core/include/treereg/*.hpp).  Each entry point below
 * names the reference declaration it replaces.  Plain pointers and sizes
 * only; all 3x3 matrices are ROW-MAJOR (the C++ adapter converts from
 * Eigen's column-major).  Every function returns a trg_status; the detail
 * string of the last failure on the calling thread is trg_last_error().
 * There is no CPU fallback: without a CUDA device every compute call
 * returns TRG_ECUDA.
 *
 * Error mapping: the reference's exception types map to
 *   std::invalid_argument      -> TRG_EINVAL
 *   std::domain_error          -> TRG_EDOMAIN
 *   std::runtime_error         -> TRG_ERUNTIME
 *   std::out_of_range          -> TRG_ERANGE
 *   DegenerateGeometryError    -> TRG_EDEGENERATE  (mstep.hpp:14-16)
 * and the adapter rethrows the same types. */
#ifndef TREEREG_B200_H
#define TREEREG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TRG_OK = 0,
  TRG_EINVAL = 1,
  TRG_EDOMAIN = 2,
  TRG_ERUNTIME = 3,
  TRG_ERANGE = 4,
  TRG_EDEGENERATE = 5,
  TRG_ECUDA = 6,
  TRG_ENCCL = 7
} trg_status;

typedef struct trg_ctx trg_ctx;           /* device, stream, workspace arena */
typedef struct trg_tree_dev trg_tree_dev; /* device-resident GMM tree */

/* treereg::ModelConfig, gmm.hpp:34-41 */
typedef struct {
  int em_iterations_per_node;        /* 8 */
  size_t min_points_per_node;        /* 32 */
  double cov_regularization_epsilon; /* 1e-4 */
  double cov_regularization_absolute;/* 1e-12 */
  uint64_t rng_seed;                 /* 0 (flat GMM only) */
  int max_level;                     /* 3 */
} trg_model_config;

/* treereg::AssocConfig, association.hpp:34-40 */
typedef struct {
  double lambda_c;      /* 0.01, in [0, 1/3] */
  int max_level;        /* 0 = full tree depth */
  double outlier_floor; /* 1e-300 */
  int deterministic;    /* kept for interface parity; always deterministic */
} trg_assoc_config;

/* treereg::Variant::Kind, registration.hpp:19-20 */
enum { TRG_VARIANT_ADAPTIVE = 0, TRG_VARIANT_TREE = 1, TRG_VARIANT_FLAT = 2, TRG_VARIANT_ICP = 3 };

/* treereg::RegistrationConfig, registration.hpp:27-36 */
typedef struct {
  int variant_kind;        /* TRG_VARIANT_ADAPTIVE | TRG_VARIANT_TREE | TRG_VARIANT_FLAT | TRG_VARIANT_ICP */
  int variant_param;       /* tree depth L */
  double lambda_c;         /* 0.01 */
  int max_em_iterations;   /* 50 */
  double rotation_tol;     /* 1e-5 rad */
  double translation_tol;  /* 1e-5 (fraction of target bbox diagonal) */
  double initial_R[9];     /* identity */
  double initial_t[3];     /* zero */
  trg_model_config model_config;
  /* Not in the reference (0 there, the parity mode): 1 = the EM's
   * association scores in FP32 (SURVEY 7.2 fast path; adaptive:L / tree:L
   * only): the point-minus-mean differences stay FP64, the quadratic form,
   * log-scores and normalisation are FP32, the deposits FP64.  Stop nodes can
   * differ from the reference's where the top two sibling log-scores are
   * within ~1e-5; transforms agree within the north_star tolerance. */
  int fast_scoring;
} trg_reg_config;

/* Host-side tree: treereg::GmmTree (gmm.hpp:56-67) + cached eigen data of
 * each GaussianComponent (gmm.hpp:12-23).  Arrays are caller-allocated with
 * `capacity` >= trg_tree_capacity(max_level) nodes. */
typedef struct {
  int n_nodes, max_level, capacity;
  double* weight;   /* [J] */
  double* mean;     /* [J*3] */
  double* cov;      /* [J*9] row-major */
  double* lambdas;  /* [J*3] descending */
  double* axes;     /* [J*9] row-major; column l = unit axis for lambdas[l] */
  double* log_norm; /* [J] */
  int* parent;      /* [J] -1 for level 0 */
  int* first_child; /* [J] -1 for leaves */
  int* child_count; /* [J] */
  int* level;       /* [J] */
} trg_tree;

/* treereg::MomentSet, association.hpp:14-32 (m1 [J*3], m2 [J*9] or NULL) */
typedef struct {
  double* m0;
  double* m1;
  double* m2;
  uint64_t total_points;
  uint64_t outliers;
  uint64_t density_evaluations;
  double total_mass;
} trg_moments;

/* treereg::BuildDiagnostics (gmm.hpp:43-49) + the device counters that
 * define the roofline bytes. */
typedef struct {
  uint64_t entries_per_round[8]; /* E_l */
  int expanded_per_round[8];
  int calibration_passes;
  double calibration_drift;
  uint64_t calib_density_evaluations;
  /* node_ll_traces (gmm.hpp:45): the kept fit's EM log-likelihoods per
   * expansion in build order, em_iterations_per_node + 1 values each.
   * Caller-allocated [ll_trace_capacity][em_iterations_per_node + 1], or NULL. */
  double* ll_traces;
  int ll_trace_capacity;
  int n_expansions;
  /* trg_build_flat_gmm only: the flat fit's per-iteration log-likelihoods
   * (gmm.cpp:729-734, em_iterations_per_node * max_level values) are written
   * contiguously at ll_traces when ll_trace_capacity *
   * (em_iterations_per_node + 1) holds them; their count goes here. */
  int flat_trace_len;
} trg_build_diag;

/* treereg::MStepSolution, mstep.hpp:54-61 */
typedef struct {
  double omega[3];
  double translation[3];
  double delta_R[9];
  double delta_t[3];
  double criterion_before;
  double criterion_after;
  double condition_estimate;
  int n_virtual_points;
} trg_mstep_solution;

/* treereg::RegistrationResult, registration.hpp:38-48.  Trace arrays are
 * caller-allocated with `trace_capacity` >= max_em_iterations (or NULL). */
typedef struct {
  double R[9];
  double t[3];
  int iterations;
  int converged;
  double* criterion_trace;
  double* criterion_after_trace;
  uint64_t* eval_counts;
  int trace_capacity;
  double model_build_seconds;
  double em_seconds;
  size_t model_components;
} trg_reg_result;

/* ---- context ---------------------------------------------------------- */
int trg_ctx_create(int device, trg_ctx** out);
int trg_ctx_destroy(trg_ctx* ctx);
const char* trg_last_error(void);
int trg_device_sms(trg_ctx* ctx);
/* Limits this context's persistent grids to `sms` SMs' worth of CTAs (0 =
 * the whole device).  Several contexts on one device, each on its own
 * stream and host thread, then run independent registrations concurrently
 * (batched frame pairs, BASELINE config C5).  No reference counterpart. */
int trg_ctx_set_sm_budget(trg_ctx* ctx, int sms);
/* Launch count of this library's kernels since ctx creation (bench evidence). */
uint64_t trg_kernel_launches(trg_ctx* ctx);
/* Bytes copied host->device / device->host by this context so far. */
void trg_ctx_transfer_bytes(trg_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* CUDA stream (cudaStream_t) all work of this context is ordered on. */
void* trg_ctx_stream(trg_ctx* ctx);
/* Orders this context's stream after the work queued so far on `stream`
 * (a cudaStream_t of the caller, e.g. the one that produced a device cloud
 * passed with *_on_device = 1).  Device inputs must be complete -- or their
 * producer's stream handed here -- before a call reads them. */
int trg_ctx_wait_stream(trg_ctx* ctx, void* stream);

/* ---- model ------------------------------------------------------------ */
int trg_tree_capacity(int max_level);
/* Upload a host tree (e.g. a load_tree() result, gmm.cpp:798-896). */
int trg_tree_upload(trg_ctx* ctx, const trg_tree* host, trg_tree_dev** out);
/* load_tree's model from its JSON fields (gmm.cpp:798-896): weight, mean,
 * cov and the topology are read from `host`; lambdas / axes / log_norm are
 * ignored and recomputed on the device (refresh_eig, gmm.cpp:31-35, for every
 * node).  TRG_EINVAL when eig_sym3 rejects a covariance, TRG_EDOMAIN when one
 * is not positive definite (the lowest such node decides, like the
 * reference's in-order loop). */
int trg_tree_upload_refresh(trg_ctx* ctx, const trg_tree* host, trg_tree_dev** out);
int trg_tree_download(trg_ctx* ctx, const trg_tree_dev* tree, trg_tree* host);
/* treereg::save_tree / load_tree (gmm.cpp:769-896): the reference's JSON
 * model file ("gmm-tree" v1), written with the reference's JSON library so
 * the bytes match.  Bad files return TRG_ERUNTIME with the reference's
 * "bad model file <path>: ..." message; a covariance eig_sym3 rejects,
 * TRG_EINVAL.  trg_load_tree computes every node's eigen fields on the
 * device (trg_tree_upload_refresh). */
int trg_save_tree(trg_ctx* ctx, const trg_tree_dev* tree, const char* path);
int trg_load_tree(trg_ctx* ctx, const char* path, trg_tree_dev** out);
/* Host halves (no device): save from / parse into a host tree.  Parse with
 * host->capacity < nodes returns TRG_ERANGE and sets host->n_nodes to the
 * size needed (lambdas / axes / log_norm are not touched). */
int trg_save_tree_host(const trg_tree* host, const char* path);
int trg_load_tree_host(const char* path, trg_tree* host);
int trg_tree_free(trg_ctx* ctx, trg_tree_dev* tree);
int trg_tree_size(const trg_tree_dev* tree);

/* treereg::build_tree (gmm.hpp:69-70).  `xyz` is N*3 AoS doubles on the host
 * (xyz_on_device = 0) or in device memory (1). */
int trg_build_tree(trg_ctx* ctx, const double* xyz, size_t n, int xyz_on_device,
                   const trg_model_config* cfg, trg_tree_dev** out, trg_build_diag* diag);

/* ---- E-step ----------------------------------------------------------- */
/* treereg::associate_adaptive (association.hpp:54-56).  Moments are written
 * to host memory.  point_node / point_weight (nullable, host, [N]) receive
 * each point's deposit node (-1 = outlier) and path weight. */
int trg_associate(trg_ctx* ctx, const trg_tree_dev* tree, const double* xyz, size_t n,
                  int xyz_on_device, const double R[9], const double t[3],
                  const trg_assoc_config* cfg, trg_moments* out, int* point_node,
                  double* point_weight);

/* ---- flat mixture ("GMM J=n") --------------------
 * treereg::build_flat_gmm (gmm.hpp:74-76, gmm.cpp:659-736): list_moments,
 * D^2-weighted seeding from mt19937_64(cfg->rng_seed) (the reference's
 * stream and libstdc++ distributions, reproduced on the device), J
 * components at sigma^2 I, em_iterations_per_node * max_level EM
 * iterations.  The mixture comes back as a depth-1 "tree" of J roots (all
 * leaves), so trg_tree_download / trg_responsibilities_dense / the EM loop
 * take it as is.  diag: entries_per_round[0] = N; no ll traces. */
int trg_build_flat_gmm(trg_ctx* ctx, const double* xyz, size_t n, int xyz_on_device, size_t J,
                       const trg_model_config* cfg, trg_tree_dev** out, trg_build_diag* diag);
/* treereg::responsibilities_dense (association.hpp:44-47, association.cpp:54-89):
 * every node of `comps` is a component (a flat mixture, or a tree's nodes).
 * Moments as trg_associate (m2 when out->m2 != NULL). */
int trg_responsibilities_dense(trg_ctx* ctx, const trg_tree_dev* comps, const double* xyz,
                               size_t n, int xyz_on_device, const double R[9], const double t[3],
                               double outlier_floor, trg_moments* out);

/* ---- M-step ----------------------------------------------------------- */
/* treereg::make_virtual_points + treereg::solve_mstep (mstep.hpp:46-47, 67)
 * on a host MomentSet (m0 [J], m1 [J*3]).  Returns TRG_EDEGENERATE where
 * the reference throws DegenerateGeometryError. */
int trg_solve_mstep(trg_ctx* ctx, const trg_tree_dev* tree, const double* m0, const double* m1,
                    uint64_t total_points, trg_mstep_solution* out);

/* treereg::make_virtual_points (mstep.hpp:46-47) on the device: the ordered
 * list of components with m0 > 1e-8 N: index[], pi* = m0/N, mu* = m1/m0
 * (arrays sized n_components; *n_out receives the count). */
int trg_make_virtual_points(trg_ctx* ctx, int n_components, const double* m0, const double* m1,
                            uint64_t total_points, int* index, double* pi_star, double* mu_star,
                            int* n_out);
/* treereg::solve_mstep(const VirtualPointSet&) (mstep.hpp:67) on explicit
 * virtual points and their components (mean [n*3], lambdas [n*3] descending,
 * axes [n*9] row-major, column l = axis of lambdas[l]). */
int trg_solve_mstep_vps(trg_ctx* ctx, int n_vps, const double* pi_star, const double* mu_star,
                        const double* comp_mean, const double* comp_lambdas,
                        const double* comp_axes, trg_mstep_solution* out);

/* ---- driver ----------------------------------------------------------- */
/* treereg::register_with_tree (registration.hpp:59-62). */
int trg_register_with_tree(trg_ctx* ctx, const trg_tree_dev* tree, const double* xyz, size_t n,
                           int xyz_on_device, const trg_reg_config* cfg, double target_diag,
                           trg_reg_result* out);
/* treereg::register_clouds (registration.hpp:53-55), adaptive:L / tree:L. */
int trg_register_clouds(trg_ctx* ctx, const double* target, size_t n_target, const double* source,
                        size_t n_source, int on_device, const trg_reg_config* cfg,
                        trg_reg_result* out);
/* Batch of independent frame pairs (BASELINE config C5).  No reference
 * counterpart: the reference registers one pair per register_clouds call
 * (registration.hpp:53-55) and a caller loops; this entry point is that
 * loop.  Pair i registers sources[i] (n_sources[i] points) to targets[i]
 * with `cfg` and fills out[i] (trace pointers as in trg_reg_result, may be
 * NULL).  Tree variants (adaptive / tree): `streams` = pairs in flight
 * (1..24; 0 = 24); the pairs run in waves, each wave's tree builds as ONE
 * cooperative launch (one CTA group per pair, group barriers) and its EM
 * loops as one more.  Flat / ICP variants: `streams` pairs (1..16; 0 = 4)
 * run concurrently, each on its own worker thread, CUDA stream and
 * 1/streams of the SMs.  Either way every pair's result is bit-identical to
 * trg_register_clouds on that pair.  Returns TRG_OK or the status of the
 * lowest-index failing pair (out[] of the others is filled). */
int trg_register_batch(trg_ctx* ctx, int n_pairs, const double* const* targets,
                       const size_t* n_targets, const double* const* sources,
                       const size_t* n_sources, int on_device, const trg_reg_config* cfg,
                       int streams, trg_reg_result* out);

/* ---- synthetic frames on the device (no reference
 *      counterpart: the C2 / C3 / C5 generators are new).  The ray casting
 *      of trg_synth_kinect_pair / trg_synth_lidar_pair (libtrg_host.so) as
 *      one thread per pixel / beam, from the poses, noise draws and beam
 *      directions trg_synth_*_pair_plan returns: bit-identical frames.
 *      R, t: frames x 9 / 3 host doubles (sensor -> world); noise: frames x
 *      76,800 (Kinect, scaled by noise_scale x the axial sigma) resp. frames
 *      x 72,000 (LiDAR, x 0.02 m) host doubles, or NULL for noise-free
 *      frames; dir_tables: 4,564 host doubles; out: DEVICE buffer of frames
 *      x points x 3 doubles, written in order on ctx's stream. */
int trg_render_kinect_frames(trg_ctx* ctx, int frames, const double* R, const double* t,
                             const double* noise, double noise_scale, double* out);
int trg_render_lidar_frames(trg_ctx* ctx, int frames, const double* R, const double* t,
                            const double* noise, const double* dir_tables, double* out);

/* ---- point-sharded execution (no reference counterpart:
 *      the reference is single-process).  A large cloud is split into
 *      contiguous blocks, one per shard; entries never move between shards.
 *      Every per-node reduction of the build (phase records), of the leaf
 *      calibration (leaf moments) and of the EM loop (per-node m0/m1) is
 *      all-reduced between kernel segments; argmax seeds (heaviest entry,
 *      farthest points) are all-gathered and resolved to the lowest global
 *      position.  Every shard then computes the same node updates, so the
 *      tree and the transform agree across shards without a broadcast.
 *      Results match the single-GPU path within the north_star tolerances
 *      (sums regroup across shards). ------------------------------------- */
typedef struct trg_comm trg_comm;
/* NCCL unique id (128 bytes) for rank 0 to share with the other ranks. */
int trg_comm_unique_id(unsigned char id[128]);
/* One shard per process over NCCL (libnccl.so.2 bound at run time). */
int trg_comm_create_nccl(trg_ctx* ctx, const unsigned char id[128], int rank, int world,
                         trg_comm** out);
/* `shards` (1..16) shards driven by this process on ctx's device, exchanged
 * by a fixed-order device reduction: the sharded algorithm on one GPU. */
int trg_comm_create_local(trg_ctx* ctx, int shards, trg_comm** out);
int trg_comm_destroy(trg_comm* comm);
int trg_comm_rank(trg_comm* comm);
int trg_comm_world(trg_comm* comm);
int trg_comm_local_shards(trg_comm* comm);
/* build_tree over the union of the shards' clouds: xyz[i] / n[i] for each of
 * the comm's local shards (one entry in NCCL mode).  Every shard gets the
 * same tree; *out is the first local shard's (on ctx's device).  diag:
 * entries_per_round summed over all shards. */
int trg_build_tree_sharded(trg_comm* comm, const double* const* xyz, const size_t* n,
                           int on_device, const trg_model_config* cfg, trg_tree_dev** out,
                           trg_build_diag* diag);
/* register_clouds over sharded target and source clouds (adaptive:L /
 * tree:L): sharded build, global bounding-box diagonal, sharded EM. */
int trg_register_clouds_sharded(trg_comm* comm, const double* const* target,
                                const size_t* n_target, const double* const* source,
                                const size_t* n_source, int on_device, const trg_reg_config* cfg,
                                trg_reg_result* out);

/* ---- host-side data: cloud ingest and the synthetic generators live in
 *      the HOST library libtrg_host.so (include/treereg_b200_host.h); the
 *      product library holds only the device path. -------------------- */

/* ---- diagnostics ------------------------------------------------------
 * Runs the device eigensolvers on `count` row-major matrices: n = 6 is the
 * 6x6 Jacobi of solve_mstep (mstep.cpp:77), n = 3 eig_sym3
 * (geometry.cpp:40-79), n = -3 eig_sym3_floored at 1e-4 (:81-102).  Used by
 * the tests to pin device math bit-for-bit to the CPU oracle. */
/* Device timeline of the last trg_build_tree on this context: globaltimer
 * (ns) at each grid barrier and a phase label (round*100 + phase; +50 for
 * the node-reduction half; 900-902 rematch; 1000+10*pass+stage calibration).
 * Returns the number of marks. */
int trg_debug_build_timeline(trg_ctx* ctx, uint64_t* t_ns, int* labels, int cap);
int trg_debug_eig(trg_ctx* ctx, int n, const double* in, int count, double* evals,
                  double* evecs, int* status);
/* Runs the device warp-level 6-DoF solve (mstep.cpp:76-98) on packed normal
 * equations v27 = (upper-triangular ata[21], atb[6]); out16 receives
 * omega[3], translation[3], condition estimate, degenerate flag. */
int trg_debug_solve(trg_ctx* ctx, const double* v27, int n_virtual_points, double* out16);

#ifdef __cplusplus
}
#endif
#endif /* TREEREG_B200_H */
