/* TEST INFRASTRUCTURE ONLY — CPU oracle, never linked into the product.
 *
 * Plain-C restatement of the reference hot path (treereg, /root/reference):
 *   trgo_build_tree          gmm.cpp:584-657 (+ helpers 31-580)
 *   trgo_associate           association.cpp:91-157
 *   trgo_solve_mstep         mstep.cpp:8-99
 *   trgo_register_with_tree  registration.cpp:47-82, 140-172
 * Arithmetic follows the reference expression by expression in the
 * evaluation order of the test Eigen shim (oracle/shim/Eigen/Core), so the
 * port is pinned bit-for-bit against oracle/_ref/libtreereg_ref.so by
 * tests/test_oracle_port.py.  Single-threaded, but merges per-4096 chunk
 * partials in chunk order exactly like parallel::for_chunks
 * (parallel.hpp:30-33), which makes results thread-count independent.
 * Matrices are ROW-MAJOR at this interface. */
#ifndef TRG_ORACLE_H
#define TRG_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int n_nodes, max_level, capacity;
  double *weight, *mean, *cov, *lambdas, *axes, *log_norm; /* axes row-major, columns = eigvecs */
  int *parent, *first_child, *child_count, *level;
} trgo_tree;

typedef struct {
  int max_level;              /* gmm.hpp:40 */
  int em_iterations_per_node; /* gmm.hpp:35 */
  size_t min_points_per_node; /* gmm.hpp:36 */
  double eps;                 /* cov_regularization_epsilon gmm.hpp:37 */
  double abs_floor;           /* cov_regularization_absolute gmm.hpp:38 */
} trgo_model_cfg;

typedef struct {
  uint64_t entries_per_round[8]; /* E_l: entries processed by expansion round l */
  int expanded_per_round[8];     /* nodes expanded per round */
  int calibration_passes;
  double calibration_drift;
  uint64_t calib_density_evals;
} trgo_build_stats;

int trgo_tree_alloc(trgo_tree* t, int capacity);
void trgo_tree_free(trgo_tree* t);
int trgo_tree_capacity(int max_level);

/* Returns 0 on success, nonzero TRG_E* code (1 invalid, 2 domain, 3 runtime). */
int trgo_build_tree(const double* xyz, size_t n, const trgo_model_cfg* cfg, trgo_tree* out,
                    trgo_build_stats* stats);

int trgo_associate(const trgo_tree* t, const double* xyz, size_t n, const double* R,
                   const double* tr, double lambda_c, int max_level, double* m0, double* m1,
                   double* m2, uint64_t* counters /*total, outliers, evals*/, double* total_mass,
                   int* point_node /*nullable*/, double* point_weight /*nullable*/);

int trgo_solve_mstep(const trgo_tree* t, const double* m0, const double* m1, uint64_t total_points,
                     double* omega, double* trans, double* dR, double* dt,
                     double* scal /*crit_before, crit_after, cond*/, int* n_vps);

int trgo_register_with_tree(const trgo_tree* t, const double* xyz, size_t n, int tree_variant,
                            double lambda_c, int max_iters, double rot_tol, double trans_tol,
                            double target_diag, double* R, double* tr, int* iters, int* converged,
                            double* crit_before, double* crit_after, uint64_t* evals);

int trgo_eig_sym3(const double* m, int floored, double floor_value, double* lambdas, double* axes);
double trgo_bbox_diagonal(const double* xyz, size_t n);
const char* trgo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
