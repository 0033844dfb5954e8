/* apb.h - C ABI of the B200-native ball dot product / block ball matmul.
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `apball` (/root/reference/proj).  Every entry point below replaces one C++
 * operator of the reference; the replaced interface is cited as file:line
 * relative to /root/reference/proj.  No C++ or torch types cross this
 * boundary: plain pointers, sizes and a cudaStream_t passed as void*.
 *
 * Data layout ("ball array", SoA, same layout on host and device):
 *   mant    uint64[count * L]  mantissa limbs of element e at mant[e*L .. e*L+L),
 *                              little-endian and TOP-ALIGNED: an ApFloat with n
 *                              limbs occupies slots L-n .. L-1, lower slots are 0.
 *                              (ApFloat keeps the minimal limb count,
 *                              include/apball/apfloat.hpp:4-9, so n is recovered
 *                              exactly as L minus the number of zero low slots.)
 *   exp     int64[count]       ApFloat exponent e: 2^(e-1) <= |x| < 2^e
 *   kind    uint8[count]       APB_ZERO/APB_FINITE/APB_PINF/APB_NINF/APB_NAN,
 *                              bit 7 (APB_SIGN) = negative finite midpoint
 *   rad_man uint32[count]      Mag mantissa b in [2^29, 2^30) (include/apball/mag.hpp:15-59);
 *                              0 = exact (zero radius), APB_RAD_INF = infinite radius
 *   rad_exp int64[count]       Mag exponent f: radius = b * 2^(f-30)
 *
 * Status codes map to the reference's exceptions:
 *   0 ok, 1 std::invalid_argument (dimensions), 2 std::overflow_error
 *   (exponent range, src/apfloat.cpp:18-22), 3 unsupported, 4 CUDA error.
 */
#ifndef APB_H
#define APB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    APB_ZERO = 0,
    APB_FINITE = 1,
    APB_PINF = 2,
    APB_NINF = 3,
    APB_NAN = 4,
    APB_KIND_MASK = 7,
    APB_SIGN = 0x80
};
#define APB_RAD_INF 0xFFFFFFFFu

enum {
    APB_OK = 0,
    APB_ERR_INVALID = 1,
    APB_ERR_OVERFLOW = 2,
    APB_ERR_UNSUPPORTED = 3,
    APB_ERR_CUDA = 4
};

typedef struct apb_balls {
    uint64_t* mant;
    int64_t* exp;
    uint8_t* kind;
    uint32_t* rad_man;
    int64_t* rad_exp;
    int64_t count;
    int32_t L;
} apb_balls;

/* Term addressing for a batch of dot products.  Dot b (0 <= b < batch) reads
 * term i (0 <= i < n) of x at element
 *     (b / bdiv) * xs1 + (b % bdiv) * xs2 + i * xstep  (+ x_off)
 * and likewise for y.  A flat batch of contiguous dots uses bdiv = 1,
 * xs1 = n, xs2 = 0, xstep = 1; a classical matmul C = A B uses bdiv = N,
 * xs1 = K, xs2 = 0, xstep = 1 and ys1 = 0, ys2 = 1, ystep = N
 * (src/matmul.cpp:442-451).  Steps may be negative (src/dot.cpp:29-43). */
typedef struct apb_dot_index {
    int64_t bdiv;
    int64_t x_off, xs1, xs2, xstep;
    int64_t y_off, ys1, ys2, ystep;
} apb_dot_index;

enum { APB_DOT_BALL = 0, APB_DOT_APPROX = 1 };

/* Dot plan + accumulator as the reference exposes them for parity
 * (include/apball/dot.hpp:25-43).  One record per dot. */
typedef struct apb_dot_state {
    int64_t e_max, e_min, e_rad;
    uint64_t n_nonzero;
    int64_t p_eff;
    int32_t extend, padding;
    int64_t n_s;
    int64_t e_s;
    int32_t status; /* 0 Proceed, 1 Fallback, 2 ZeroResult (DotStatus) */
    int32_t _pad;
    uint64_t err;
    uint64_t srad;
} apb_dot_state;

/* Device-side tuning knobs mirrored from DotTuning (include/apball/dot.hpp:45-51). */
typedef struct apb_dot_tuning {
    int32_t disable_precision_reduction;
    int32_t force_threeprod;
    int64_t threeprod_cutoff_limbs;
} apb_dot_tuning;

/* ------------------------------------------------------------------ dots */

/* Batched real ball / approx dot product, all pointers DEVICE.
 * Replaces dot_ball (include/apball/dot.hpp:73-74, src/dot.cpp:402-405) and
 * dot_approx (dot.hpp:77-78) called once per dot.  `initial` (nullable) holds
 * one ball per dot (element b), `subtract` negates the sum.  out must have
 * L >= ceil(prec/64) and count >= batch.  mode = APB_DOT_BALL|APB_DOT_APPROX
 * (approx writes zero radii).  state (nullable, device) receives the plan and
 * the final accumulator scalars per dot; acc_limbs (nullable, device) receives
 * n_s two's-complement accumulator limbs per dot at stride acc_stride (the
 * state BEFORE dot_finalize), for bit-exact parity with dot_setup/dot_init/
 * dot_accumulate_term (dot.hpp:57-69). */
int apb_dot_batch(const apb_balls* x, const apb_balls* y, const apb_balls* initial,
                  int subtract, const apb_dot_index* idx, int64_t n, int64_t batch,
                  int64_t prec, int mode, const apb_dot_tuning* tuning, apb_balls* out,
                  apb_dot_state* state, uint64_t* acc_limbs, int64_t acc_stride,
                  void* stream);

/* Batched complex dot product (re/im as two ball arrays per operand), DEVICE.
 * Replaces dot_complex_ball / dot_complex_approx (include/apball/dot.hpp:86-89,
 * src/dot.cpp:549-568).  threeprod_hits (nullable, device uint64[1]) is
 * incremented like dot_threeprod_hits() (dot.hpp:54). */
int apb_dot_complex_batch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                          const apb_balls* yim, const apb_dot_index* idx, int64_t n,
                          int64_t batch, int64_t prec, int mode, const apb_dot_tuning* tuning,
                          apb_balls* out_re, apb_balls* out_im, uint64_t* threeprod_hits,
                          void* stream);

/* ---------------------------------------------------------------- matmul */

typedef struct apb_mat {
    apb_balls b; /* rows*cols balls, row-major (include/apball/matmul.hpp:18-26) */
    int64_t rows, cols;
} apb_mat;

enum { APB_MM_AUTO = 0, APB_MM_BLOCK = 1, APB_MM_CLASSICAL = 2 };

/* Matmul statistics mirrored from MatmulStats (include/apball/matmul.hpp:98-105);
 * int_gemm_products counts scaled-integer GEMMs run on the tensor cores
 * (the reference counts multimodular products instead). */
typedef struct apb_matmul_stats {
    uint64_t classical_calls;
    uint64_t block_calls;
    uint64_t int_gemm_products;
    uint64_t last_block_count;
    uint64_t last_height_a, last_height_b, last_slices_a, last_slices_b;
} apb_matmul_stats;

/* C = A B over balls, all matrices DEVICE.  Replaces matmul_auto /
 * block_matmul_ball / classical_matmul_ball (include/apball/matmul.hpp:89-91,
 * src/matmul.cpp:442-531).  C must have L >= ceil(prec/64). */
int apb_matmul(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
               void* stream);

/* Complex C = A B (re/im parts), DEVICE.  Replaces complex_matmul_ball
 * (include/apball/matmul.hpp:92-93, src/matmul.cpp:533-548): four real
 * products each rounded to prec, then re = AC - BD, im = AD + BC. */
int apb_matmul_complex(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre,
                       const apb_mat* Bim, int64_t prec, int algo, apb_mat* Cre, apb_mat* Cim,
                       void* stream);

/* Parity hook: the exact scaled-integer block product of a single block
 * [lo,hi) (matmul.hpp:77-84: int_matmul(scale_block_rows(A), scale_block_cols(B))).
 * Writes the row/col scale exponents (int64[M], int64[N], DEVICE) and the
 * exact product as little-endian two's-complement limbs, `out_limbs` limbs
 * per entry (DEVICE uint64[M*N*out_limbs]).  Returns APB_ERR_UNSUPPORTED if
 * out_limbs is too small for the product height. */
int apb_block_int_product(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi,
                          int64_t* row_scale, int64_t* col_scale, uint64_t* out,
                          int64_t out_limbs, void* stream);

/* Measurement baseline: the same exact block product as apb_block_int_product
 * computed with 32-bit limbs on the CUDA cores (IMAD.WIDE.U32, one thread per
 * output entry) instead of int8 slices on the tensor cores -- the alternative
 * the int8 design is chosen against (BASELINE.json north_star).  Same outputs;
 * *gemm_ms (nullable) receives the product kernel's time.  Heights above
 * 19 x 32 bits return APB_ERR_UNSUPPORTED.  Synchronizes the stream. */
int apb_block_int_product_imad(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi,
                               int64_t* row_scale, int64_t* col_scale, uint64_t* out,
                               int64_t out_limbs, float* gemm_ms, void* stream);

/* Parity hook: greedy block plan (include/apball/matmul.hpp:73, src/matmul.cpp:132-161).
 * steps_out receives up to max_steps triples (lo, hi, basecase); *n_steps the count. */
int apb_plan_blocks(const apb_mat* A, const apb_mat* B, int64_t prec, int64_t* steps_out,
                    int64_t max_steps, int64_t* n_steps, void* stream);

/* Parity hook: radius product upper bound of two Mag matrices given as
 * (rad_man, rad_exp) planes (include/apball/matmul.hpp:87, src/matmul.cpp:368-438). */
int apb_radius_matmul_upper(const uint32_t* p_man, const int64_t* p_exp, const uint32_t* q_man,
                            const int64_t* q_exp, int64_t m, int64_t n, int64_t k,
                            uint32_t* out_man, int64_t* out_exp, void* stream);

/* Plan summary of C = A B without computing it (the planner of
 * src/matmul.cpp:132-161 plus the radius-product windows of :386-392), used
 * by the row-block sharded driver to verify that every shard's plan is the
 * global plan (paper_1901_04289_b200/dist.py). */
typedef struct apb_plan_info {
    int64_t n_blocks;
    int64_t entry_prec_a, entry_prec_b;
    int64_t max_width_a, max_width_b;  /* widest row window of A / column window of B */
    int32_t special;                   /* non-finite input: block path = classical */
    int32_t radius_single;             /* both radius products single-block (<= 900 bits) */
} apb_plan_info;
int apb_matmul_plan_info(const apb_mat* A, const apb_mat* B, int64_t prec, apb_plan_info* out,
                         void* stream);

/* --------------------------------------------------------- host wrappers */

/* End-to-end variants taking HOST ball arrays: host->device copy, kernels,
 * device->host copy inside one call (the drop-in path for callers holding
 * host data). */
/* host-buffer form of apb_dot_complex_batch (H2D, launch, D2H); threeprod_hits
 * (nullable) is a HOST counter that receives the gate's hit count */
int apb_dot_complex_batch_host(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                               const apb_balls* yim, const apb_dot_index* idx, int64_t n, int64_t batch,
                               int64_t prec, int mode, const apb_dot_tuning* tuning, apb_balls* out_re,
                               apb_balls* out_im, uint64_t* threeprod_hits);
/* poly_mullow_classical (include/apball/poly.hpp:23-24, src/poly.cpp:11-26):
 * out[k] = sum_i a_i b_{k-i} for k < len as one batch of variable-length fused
 * ball dots (negative step on b); out needs len slots of >= ceil(prec/64) limbs. */
int apb_poly_mullow(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                    int64_t prec, apb_balls* out, void* stream);
/* series_exp_basecase (include/apball/poly.hpp:27-29, src/poly.cpp:28-46):
 * b_0 = 1, b_k = (sum_{j=1}^{k} (j a_j) b_{k-j}) / k; APB_ERR_INVALID (the
 * reference's std::domain_error) unless a_0 is an exact zero.  Sequential in k. */
int apb_series_exp(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out, void* stream);
int apb_poly_mullow_host(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                         int64_t prec, apb_balls* out);
int apb_series_exp_host(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out);

/* Text wire format of the reference on HOST ball arrays (src/apfloat.cpp:333-390,
 * src/mag.cpp:174-197, src/ball.cpp:45-56, src/matmul.cpp:552-570): one
 * "mid +- rad" line per ball, e.g. "(+,3,8000000000000000) +- (20000000,-60)".
 * The format calls return the text length (excluding the NUL) and write it when
 * cap exceeds it; parse returns the number of balls read or -1 (apb_last_error
 * names the malformed line).  Mantissas must fit the output's L slots. */
int64_t apb_balls_format(const apb_balls* a, int64_t first, int64_t count, char* buf, int64_t cap);
int64_t apb_balls_parse(const char* text, int64_t len, apb_balls* out, int64_t count);
int64_t apb_mat_format(const apb_mat* m, char* buf, int64_t cap);
int apb_mat_parse(const char* text, int64_t len, apb_mat* out);

int apb_dot_batch_host(const apb_balls* x, const apb_balls* y, const apb_balls* initial,
                       int subtract, const apb_dot_index* idx, int64_t n, int64_t batch,
                       int64_t prec, int mode, apb_balls* out);
int apb_matmul_host(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C);
int apb_matmul_complex_host(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre,
                            const apb_mat* Bim, int64_t prec, int algo, apb_mat* Cre, apb_mat* Cim);

/* Pipelined host entry for a stream of products (serving): apb_matmul_host
 * split into a submission and a drain.  Consecutive submissions alternate
 * between two device buffer sets, so the host->device copy of product i+1
 * overlaps the compute and the device->host copy of product i (three streams:
 * copy-in, compute, copy-out).  The host buffers of a submitted product
 * (pinned memory for overlap) must stay untouched until apb_matmul_host_drain
 * returns, which waits for every submitted product and returns the first error.
 * A submission returns once its copy-in is queued; a library worker thread
 * queues the product and its copy-out.  Drain before other library calls.
 * Results are identical to apb_matmul_host. */
int apb_matmul_host_submit(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C);
int apb_matmul_host_drain(void);

/* ------------------------------------------------------------------ misc */

/* Synchronize `stream` and return (then clear) the APB_* status raised by
 * device code since the last call (e.g. APB_ERR_OVERFLOW where the reference
 * throws std::overflow_error, src/apfloat.cpp:18-22).  The device entry points
 * above are asynchronous and only report launch/argument errors. */
int apb_device_status(void* stream);

/* Kernel-level timing for measurement: when enabled, the library brackets its
 * kernels with CUDA events on the launching stream, grouped by name
 * ("slice_gemm", "dot", "pack", "recombine", "rad_gemm", "scan").
 * apb_profile_read synchronizes the recorded events and returns the summed
 * device milliseconds and the number of launches since the last reset. */
void apb_profile_enable(int on);
void apb_profile_reset(void);
int apb_profile_read(const char* kernel, double* ms, uint64_t* launches);
/* timeline of every recorded region as "name<TAB>begin_ms<TAB>end_ms" lines,
 * relative to the first region's begin (regions on all streams); returns the
 * full text length (buf may be NULL to query it) */
int apb_profile_dump(char* buf, size_t cap);
/* device-side span timer of the exact-integer band GEMM (first CTA start to
 * last CTA end, ns), accumulated over launches -- also inside the library's
 * captured CUDA graphs, where per-call event regions are not recorded */
int apb_gemm_timer_read(uint64_t* total_ns, uint64_t* launches);
int apb_gemm_timer_reset(void);
/* shape of the last band GEMM launched (measurement aid): output tile width (128 / 256),
 * diagonals per band, raw-accumulator epilogue (0/1), K splits */
int apb_gemm_last_config(int* tile_n, int* band_w, int* raw, int* ksplit);

apb_matmul_stats* apb_matmul_stats_get(void);
void apb_matmul_stats_reset(void);
const char* apb_last_error(void);
/* number of kernel launches issued by this library since load (bench evidence) */
uint64_t apb_launch_count(void);
int apb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* APB_H */
