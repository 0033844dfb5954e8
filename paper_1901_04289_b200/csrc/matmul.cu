// matmul.cu - ball matrix multiplication driver (src/matmul.cpp:442-548).
// Classical path: one batched dot launch over all (i,j) (src/matmul.cpp:442-451).
#include <cuda_runtime.h>

#include "apb.h"
#include "apb_internal.h"

namespace apb {

apb_matmul_stats& stats();

static int classical(const apb_mat* A, const apb_mat* B, int64_t prec, apb_mat* C, cudaStream_t st) {
    stats().classical_calls++;
    apb_dot_index ix;
    ix.bdiv = B->cols;
    ix.x_off = 0;
    ix.xs1 = A->cols;
    ix.xs2 = 0;
    ix.xstep = 1;
    ix.y_off = 0;
    ix.ys1 = 0;
    ix.ys2 = 1;
    ix.ystep = B->cols;
    return dot_batch_launch(&A->b, &B->b, nullptr, 0, &ix, A->cols, A->rows * B->cols, prec,
                            APB_DOT_BALL, nullptr, &C->b, nullptr, nullptr, 0, st);
}

int matmul_launch(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
                  cudaStream_t st) {
    if (A->rows * B->cols == 0) return APB_OK;
    if (A->cols == 0 || algo == APB_MM_CLASSICAL) return classical(A, B, prec, C, st);
    set_error("block matmul not built yet");
    return APB_ERR_UNSUPPORTED;
}

}  // namespace apb

extern "C" {
int apb_matmul_complex(const apb_mat*, const apb_mat*, const apb_mat*, const apb_mat*, int64_t, int,
                       apb_mat*, apb_mat*, void*) {
    apb::set_error("complex matmul not built yet");
    return APB_ERR_UNSUPPORTED;
}
int apb_block_int_product(const apb_mat*, const apb_mat*, int64_t, int64_t, int64_t*, int64_t*,
                          uint64_t*, int64_t, void*) {
    apb::set_error("not built yet");
    return APB_ERR_UNSUPPORTED;
}
int apb_plan_blocks(const apb_mat*, const apb_mat*, int64_t, int64_t*, int64_t, int64_t*, void*) {
    apb::set_error("not built yet");
    return APB_ERR_UNSUPPORTED;
}
int apb_radius_matmul_upper(const uint32_t*, const int64_t*, const uint32_t*, const int64_t*, int64_t,
                            int64_t, int64_t, uint32_t*, int64_t*, void*) {
    apb::set_error("not built yet");
    return APB_ERR_UNSUPPORTED;
}
}
