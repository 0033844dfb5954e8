/* apb_oracle.h - TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference algorithms on the hot path (ball dot product, block ball matmul).
 *
 * This is the CHECKER, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  Each function cites the
 * reference file:line (relative to /root/reference/proj) it restates.
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libapball_ref.so built from the reference sources) and the
 * committed golden fixtures in tests/golden (tests/test_oracle_golden.py).
 *
 * Data layout: the SoA ball arrays of include/apb.h.
 */
#ifndef APB_ORACLE_H
#define APB_ORACLE_H
#include "apb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* dot_ball / dot_approx per dot (src/dot.cpp:361-410); state (nullable)
 * receives the plan and err/srad, acc (nullable) the n_s accumulator limbs
 * before finalize.  Returns an APB_* status. */
int orc_dot_batch(const apb_balls* x, const apb_balls* y, const apb_balls* initial, int subtract,
                  const apb_dot_index* idx, int64_t n, int64_t batch, int64_t prec, int mode,
                  int disable_reduction, apb_balls* out, apb_dot_state* state, uint64_t* acc,
                  int64_t acc_stride);

/* dot_complex_ball / _approx without the (result-neutral) 3-mult rewrite
 * (src/dot.cpp:470-568) */
int orc_dot_complex_batch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                          const apb_balls* yim, const apb_dot_index* idx, int64_t n,
                          int64_t batch, int64_t prec, int mode, apb_balls* ore, apb_balls* oim);

/* matmul_auto / block / classical (src/matmul.cpp:442-531) */
int orc_poly_mullow(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                    int64_t prec, apb_balls* out);
int orc_series_exp(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out);
int orc_matmul(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
               int64_t* block_count);
int orc_matmul_complex(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre,
                       const apb_mat* Bim, int64_t prec, apb_mat* Cre, apb_mat* Cim);

/* plan_blocks (src/matmul.cpp:132-161): triples (lo, hi, basecase) */
int orc_plan_blocks(const apb_mat* A, const apb_mat* B, int64_t prec, int64_t* steps,
                    int64_t max_steps, int64_t* n_steps);

/* int_matmul(scale_block_rows, scale_block_cols) of one block as two's
 * complement limbs (include/apball/matmul.hpp:77-84) */
int orc_block_int_product(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi,
                          int64_t* row_scale, int64_t* col_scale, uint64_t* out,
                          int64_t out_limbs);

/* radius_matmul_upper (src/matmul.cpp:368-438) */
int orc_radius_matmul_upper(const uint32_t* pm, const int64_t* pe, const uint32_t* qm,
                            const int64_t* qe, int64_t m, int64_t n, int64_t k, uint32_t* om,
                            int64_t* oe);

#ifdef __cplusplus
}
#endif
#endif
