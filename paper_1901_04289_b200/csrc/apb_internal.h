// apb_internal.h - host-side internals shared by the translation units of
// libapb_b200.so: workspace (device scratch + status word), launch counter,
// error reporting and the kernel launchers.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

#include "apb.h"

namespace apb {

// Device scratch owned by the library, grown on demand.  Slot `k` is an
// independent buffer; the status word collects APB_ERR_* codes raised on the
// device (exponent overflow = std::overflow_error in the reference).
struct Workspace {
    int* status_dev = nullptr;
    void* bufs[96] = {};  // 64..93: the two buffer sets of the pipelined host entry
    size_t caps[96] = {};
    void* scratch(cudaStream_t st, size_t bytes, int slot);
};
Workspace& workspace();

// Library-wide serialization of the public entry points (a recursive lock; the
// pipelined host entry's worker thread takes it around each product).  A
// top-level entry first waits until every pipelined product has been enqueued
// and has finished, folding a device status raised by one of them into the
// pipeline's pending error (reported by apb_matmul_host_drain), so no other call
// can observe or clear it and no host state (workspace, scratch tables, stats,
// status word) is touched by two threads at once.
struct ApiLock {
    ApiLock();
    ~ApiLock();
    ApiLock(const ApiLock&) = delete;
    ApiLock& operator=(const ApiLock&) = delete;
    // for the pipeline itself: take the lock without waiting for the pipeline
    struct NoDrain {};
    explicit ApiLock(NoDrain);
};

void count_launch(uint64_t k = 1);
void launch_count_adjust(int64_t d);  // graph replays: kernels counted at capture, added per launch

// event-bracketed kernel timing (apb_profile_*); prof_begin returns a token
// (-1 when profiling is off) to pass to prof_end after the launch(es)
int prof_begin(const char* name, cudaStream_t st);
bool prof_enabled();
void prof_end(int token, cudaStream_t st);
void set_error(const char* msg);
int cuda_check(cudaError_t e, const char* where);

// Programmatic dependent launch: the kernel may be scheduled while its stream
// predecessor drains; it must call griddep_wait() (apb_common.cuh) before it
// reads the predecessor's output.  APB_NO_PDL=1 falls back to plain launches.
inline bool pdl_enabled() {
    static const bool on = std::getenv("APB_NO_PDL") == nullptr;
    return on;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// dot launchers (dot_kernels.cu)
int dot_batch_launch(const apb_balls* x, const apb_balls* y, const apb_balls* initial,
                     int subtract, const apb_dot_index* idx, int64_t n, int64_t batch, int64_t prec,
                     int mode, const apb_dot_tuning* tuning, apb_balls* out, apb_dot_state* state,
                     uint64_t* acc, int64_t acc_stride, cudaStream_t st);
int poly_mullow_launch(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                       int64_t prec, apb_balls* out, cudaStream_t st);
int series_exp_launch(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out,
                      cudaStream_t st);
int dot_complex_launch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                       const apb_balls* yim, const apb_dot_index* idx, int64_t n, int64_t batch,
                       int64_t prec, int mode, apb_balls* ore, apb_balls* oim, cudaStream_t st,
                       const apb_dot_tuning* tuning = nullptr, uint64_t* hits = nullptr);

// matmul launchers (matmul.cu)
int matmul_launch(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
                  cudaStream_t st);

}  // namespace apb
