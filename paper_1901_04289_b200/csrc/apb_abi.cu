// apb_abi.cu - the extern "C" boundary (include/apb.h): argument checks,
// status/error plumbing, library-owned device workspace and the host-buffer
// (end-to-end) wrappers.  The compute lives in dot_kernels.cu / matmul.cu.

#include <atomic>
#include <cstdio>
#include <cstring>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "apb.h"
#include "apb_internal.h"

namespace apb {

static std::atomic<uint64_t> g_launches{0};
static thread_local std::string g_error;
static apb_matmul_stats g_stats;

void count_launch(uint64_t k) { g_launches += k; }
void launch_count_adjust(int64_t d) { g_launches += (uint64_t)d; }
void set_error(const char* msg) { g_error = msg ? msg : ""; }

int cuda_check(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return APB_OK;
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    set_error(m.c_str());
    return APB_ERR_CUDA;
}

static std::mutex g_ws_mu;

// ---------------------------------------------------------- API lock
static std::recursive_mutex g_api_mu;
static thread_local int t_api_depth = 0;
static bool pipe_busy();
static void pipe_quiet_drain();

ApiLock::ApiLock(NoDrain) {
    g_api_mu.lock();
    t_api_depth++;
}
ApiLock::ApiLock() {
    for (;;) {
        g_api_mu.lock();
        if (t_api_depth > 0 || !pipe_busy()) break;  // nested calls never wait
        g_api_mu.unlock();
        pipe_quiet_drain();
    }
    t_api_depth++;
}
ApiLock::~ApiLock() {
    t_api_depth--;
    g_api_mu.unlock();
}

// ------------------------------------------------------------- profiling
struct ProfRec {
    std::string name;
    cudaEvent_t b, e;
    bool open;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;

bool prof_enabled() { return g_prof_on; }

int prof_begin(const char* name, cudaStream_t st) {
    if (!g_prof_on) return -1;
    std::lock_guard<std::mutex> g(g_prof_mu);
    ProfRec r;
    r.name = name;
    cudaEventCreate(&r.b);
    cudaEventCreate(&r.e);
    r.open = true;
    cudaEventRecord(r.b, st);
    g_prof.push_back(r);
    return (int)g_prof.size() - 1;
}

void prof_end(int token, cudaStream_t st) {
    if (token < 0) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (token >= (int)g_prof.size()) return;
    cudaEventRecord(g_prof[token].e, st);
    g_prof[token].open = false;
}

Workspace& workspace() {
    static Workspace* ws = [] {
        auto* w = new Workspace();
        cudaMalloc(&w->status_dev, sizeof(int));
        cudaMemset(w->status_dev, 0, sizeof(int));
        return w;
    }();
    return *ws;
}

void* Workspace::scratch(cudaStream_t st, size_t bytes, int slot) {
    std::lock_guard<std::mutex> g(g_ws_mu);
    if (bytes == 0) bytes = 1;
    if (caps[slot] < bytes) {
        if (bufs[slot]) {
            cudaStreamSynchronize(st);
            cudaFree(bufs[slot]);
        }
        size_t cap = bytes + bytes / 4 + 256;
        if (cudaMalloc(&bufs[slot], cap) != cudaSuccess) {
            bufs[slot] = nullptr;
            caps[slot] = 0;
            return nullptr;
        }
        caps[slot] = cap;
    }
    return bufs[slot];
}

apb_matmul_stats& stats() { return g_stats; }

static int64_t limbs_for(int64_t prec) { return prec <= 64 ? 1 : (prec + 63) / 64; }

static bool balls_ok(const apb_balls* a) {
    return a && a->mant && a->exp && a->kind && a->rad_man && a->rad_exp && a->L >= 1;
}

}  // namespace apb

using namespace apb;

extern "C" {

int apb_version(void) { return 1; }
uint64_t apb_launch_count(void) { return g_launches.load(); }
const char* apb_last_error(void) { return g_error.c_str(); }
apb_matmul_stats* apb_matmul_stats_get(void) {
    ApiLock api_lock;  // pending pipelined products have updated the counters
    return &g_stats;
}
void apb_matmul_stats_reset(void) {
    ApiLock api_lock;
    std::memset(&g_stats, 0, sizeof g_stats);
}

void apb_profile_enable(int on) { g_prof_on = on != 0; }

void apb_profile_reset(void) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto& r : g_prof) {
        cudaEventSynchronize(r.e);
        cudaEventDestroy(r.b);
        cudaEventDestroy(r.e);
    }
    g_prof.clear();
}

int apb_profile_read(const char* kernel, double* ms, uint64_t* launches) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    double t = 0;
    uint64_t n = 0;
    for (auto& r : g_prof) {
        if (r.open || r.name != kernel) continue;
        if (cudaEventSynchronize(r.e) != cudaSuccess) return APB_ERR_CUDA;
        float f = 0;
        cudaEventElapsedTime(&f, r.b, r.e);
        t += f;
        n++;
    }
    if (ms) *ms = t;
    if (launches) *launches = n;
    return APB_OK;
}

int apb_profile_dump(char* buf, size_t cap) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    std::string out;
    cudaEvent_t t0 = nullptr;
    for (auto& r : g_prof) {
        if (r.open) continue;
        if (cudaEventSynchronize(r.e) != cudaSuccess) return APB_ERR_CUDA;
        if (!t0) t0 = r.b;
        float b = 0, e = 0;
        cudaEventElapsedTime(&b, t0, r.b);
        cudaEventElapsedTime(&e, t0, r.e);
        char line[160];
        std::snprintf(line, sizeof line, "%s\t%.4f\t%.4f\n", r.name.c_str(), (double)b, (double)e);
        out += line;
    }
    if (buf && cap) {
        const size_t n = std::min(cap - 1, out.size());
        std::memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return (int)out.size();
}

int apb_device_status(void* stream) {
    ApiLock api_lock;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = cuda_check(cudaStreamSynchronize(st), "apb_device_status");
    if (rc) return rc;
    int h = 0;
    Workspace& ws = workspace();
    rc = cuda_check(cudaMemcpy(&h, ws.status_dev, sizeof(int), cudaMemcpyDeviceToHost), "status read");
    if (rc) return rc;
    if (h) {
        cudaMemset(ws.status_dev, 0, sizeof(int));
        set_error(h == APB_ERR_OVERFLOW ? "apball: exponent out of representable range"
                                        : "device-side error");
    }
    return h;
}

int apb_dot_batch(const apb_balls* x, const apb_balls* y, const apb_balls* initial, int subtract,
                  const apb_dot_index* idx, int64_t n, int64_t batch, int64_t prec, int mode,
                  const apb_dot_tuning* tuning, apb_balls* out, apb_dot_state* state,
                  uint64_t* acc_limbs, int64_t acc_stride, void* stream) {
    ApiLock api_lock;
    if (batch < 0 || n < 0 || !idx || !out || !balls_ok(out) || idx->bdiv < 1) {
        set_error("apb_dot_batch: invalid arguments");
        return APB_ERR_INVALID;
    }
    if (n > 0 && (!balls_ok(x) || !balls_ok(y))) {
        set_error("apb_dot_batch: missing operands");
        return APB_ERR_INVALID;
    }
    if (prec < 2) prec = 2;
    if (out->L < limbs_for(prec) || out->count < batch) {
        set_error("apb_dot_batch: output slots too small for prec");
        return APB_ERR_INVALID;
    }
    if (initial && !balls_ok(initial)) {
        set_error("apb_dot_batch: bad initial");
        return APB_ERR_INVALID;
    }
    // n == 0 with no x/y: substitute the output as a never-read operand
    const apb_balls* xx = n > 0 ? x : out;
    const apb_balls* yy = n > 0 ? y : out;
    int rc = dot_batch_launch(xx, yy, initial, subtract, idx, n, batch, prec, mode, tuning, out,
                              state, acc_limbs, acc_stride, (cudaStream_t)stream);
    if (rc) return rc;
    return cuda_check(cudaGetLastError(), "apb_dot_batch launch");
}

int apb_poly_mullow(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                    int64_t prec, apb_balls* out, void* stream) {
    ApiLock api_lock;
    if (alen < 0 || blen < 0 || len < 0 || !out || !balls_ok(out) || (alen > 0 && (!balls_ok(a) || a->count < alen)) ||
        (blen > 0 && (!balls_ok(b) || b->count < blen))) {
        set_error("apb_poly_mullow: invalid arguments");
        return APB_ERR_INVALID;
    }
    if (prec < 2) prec = 2;
    if (out->L < limbs_for(prec) || out->count < len) {
        set_error("apb_poly_mullow: output slots too small for prec");
        return APB_ERR_INVALID;
    }
    const apb_balls* aa = alen > 0 ? a : out;
    const apb_balls* bb = blen > 0 ? b : out;
    int rc = poly_mullow_launch(aa, alen, bb, blen, len, prec, out, (cudaStream_t)stream);
    if (rc) return rc;
    return cuda_check(cudaGetLastError(), "apb_poly_mullow launch");
}

int apb_series_exp(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out, void* stream) {
    ApiLock api_lock;
    if (alen < 0 || len < 0 || !out || !balls_ok(out) || (alen > 0 && (!balls_ok(a) || a->count < alen))) {
        set_error("apb_series_exp: invalid arguments");
        return APB_ERR_INVALID;
    }
    if (prec < 2) prec = 2;
    if (out->L < limbs_for(prec) || out->count < len) {
        set_error("apb_series_exp: output slots too small for prec");
        return APB_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (alen > 0) {  // the constant term must be an exact zero (src/poly.cpp:29-30: std::domain_error)
        uint8_t k0 = 0;
        uint32_t r0 = 0;
        if (cudaMemcpyAsync(&k0, a->kind, 1, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaMemcpyAsync(&r0, a->rad_man, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return cuda_check(cudaGetLastError(), "apb_series_exp");
        if ((k0 & APB_KIND_MASK) != APB_ZERO || r0 != 0) {
            set_error("series_exp_basecase: constant term must be exactly zero");
            return APB_ERR_INVALID;
        }
    }
    int rc = series_exp_launch(alen > 0 ? a : out, alen, len, prec, out, st);
    if (rc) return rc;
    return cuda_check(cudaGetLastError(), "apb_series_exp launch");
}

int apb_dot_complex_batch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                          const apb_balls* yim, const apb_dot_index* idx, int64_t n, int64_t batch,
                          int64_t prec, int mode, const apb_dot_tuning* tuning, apb_balls* out_re,
                          apb_balls* out_im, uint64_t* threeprod_hits, void* stream) {
    ApiLock api_lock;
    if (batch < 0 || n < 0 || !idx || !balls_ok(out_re) || !balls_ok(out_im) || idx->bdiv < 1) {
        set_error("apb_dot_complex_batch: invalid arguments");
        return APB_ERR_INVALID;
    }
    if (n > 0 && (!balls_ok(xre) || !balls_ok(xim) || !balls_ok(yre) || !balls_ok(yim))) {
        set_error("apb_dot_complex_batch: missing operands");
        return APB_ERR_INVALID;
    }
    if (prec < 2) prec = 2;
    if (out_re->L < limbs_for(prec) || out_im->L < limbs_for(prec)) {
        set_error("apb_dot_complex_batch: output slots too small for prec");
        return APB_ERR_INVALID;
    }
    const apb_balls* a = n > 0 ? xre : out_re;
    const apb_balls* b = n > 0 ? xim : out_re;
    const apb_balls* c = n > 0 ? yre : out_re;
    const apb_balls* d = n > 0 ? yim : out_re;
    int rc = dot_complex_launch(a, b, c, d, idx, n, batch, prec, mode, out_re, out_im,
                                (cudaStream_t)stream, tuning, threeprod_hits);
    if (rc) return rc;
    return cuda_check(cudaGetLastError(), "apb_dot_complex_batch launch");
}

int apb_matmul(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
               void* stream) {
    ApiLock api_lock;
    if (!A || !B || !C) {
        set_error("apb_matmul: null matrix");
        return APB_ERR_INVALID;
    }
    if (A->cols != B->rows || C->rows != A->rows || C->cols != B->cols) {
        set_error("matmul: dimension mismatch");
        return APB_ERR_INVALID;
    }
    if (prec < 2) prec = 2;
    if (C->b.L < limbs_for(prec)) {
        set_error("apb_matmul: output slots too small for prec");
        return APB_ERR_INVALID;
    }
    int rc = matmul_launch(A, B, prec, algo, C, (cudaStream_t)stream);
    if (rc) return rc;
    return cuda_check(cudaGetLastError(), "apb_matmul launch");
}

// ---------------------------------------------------------- host wrappers

namespace {

struct DevBalls {
    apb_balls d;
};

// copy a host ball array into workspace slots [slot0, slot0+5)
// the five SoA arrays of a ball array, one asynchronous copy each
int copy_arrays(const apb_balls* dst, const apb_balls* src, cudaMemcpyKind kind, cudaStream_t st) {
    const size_t cnt = (size_t)src->count;
    void* dsts[5] = {dst->mant, dst->exp, dst->kind, dst->rad_man, dst->rad_exp};
    void* srcs[5] = {src->mant, src->exp, src->kind, src->rad_man, src->rad_exp};
    size_t sizes[5] = {cnt * src->L * 8, cnt * 8, cnt, cnt * 4, cnt * 8};
    for (int f = 0; f < 5; f++) cudaMemcpyAsync(dsts[f], srcs[f], sizes[f], kind, st);
    return 0;
}

int to_device(const apb_balls* h, apb_balls* d, int slot0, cudaStream_t st, bool copy) {
    Workspace& ws = workspace();
    const size_t cnt = (size_t)h->count;
    d->count = h->count;
    d->L = h->L;
    d->mant = (uint64_t*)ws.scratch(st, cnt * h->L * 8, slot0);
    d->exp = (int64_t*)ws.scratch(st, cnt * 8, slot0 + 1);
    d->kind = (uint8_t*)ws.scratch(st, cnt, slot0 + 2);
    d->rad_man = (uint32_t*)ws.scratch(st, cnt * 4, slot0 + 3);
    d->rad_exp = (int64_t*)ws.scratch(st, cnt * 8, slot0 + 4);
    if (!d->mant || !d->exp || !d->kind || !d->rad_man || !d->rad_exp) {
        set_error("out of device memory");
        return APB_ERR_CUDA;
    }
    if (!copy || cnt == 0) return APB_OK;
    return copy_arrays(d, h, cudaMemcpyHostToDevice, st) ? APB_ERR_CUDA : cuda_check(cudaGetLastError(), "h2d");
}

int to_host(const apb_balls* d, apb_balls* h, cudaStream_t st) {
    const size_t cnt = (size_t)h->count;
    if (cnt == 0) return APB_OK;
    return copy_arrays(h, d, cudaMemcpyDeviceToHost, st) ? APB_ERR_CUDA : cuda_check(cudaGetLastError(), "d2h");
}

cudaStream_t host_stream() {
    static cudaStream_t s = [] {
        cudaStream_t t;
        cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
        return t;
    }();
    return s;
}

}  // namespace

int apb_dot_batch_host(const apb_balls* x, const apb_balls* y, const apb_balls* initial,
                       int subtract, const apb_dot_index* idx, int64_t n, int64_t batch,
                       int64_t prec, int mode, apb_balls* out) {
    ApiLock api_lock;
    cudaStream_t st = host_stream();
    apb_balls dx{}, dy{}, di{}, dout{};
    int rc;
    if (n > 0) {
        if ((rc = to_device(x, &dx, 5, st, true))) return rc;
        if ((rc = to_device(y, &dy, 10, st, true))) return rc;
    }
    if (initial && (rc = to_device(initial, &di, 15, st, true))) return rc;
    apb_balls hout = *out;
    hout.count = batch;
    if ((rc = to_device(&hout, &dout, 0, st, false))) return rc;
    rc = apb_dot_batch(n > 0 ? &dx : nullptr, n > 0 ? &dy : nullptr, initial ? &di : nullptr,
                       subtract, idx, n, batch, prec, mode, nullptr, &dout, nullptr, nullptr, 0, st);
    if (rc) return rc;
    if ((rc = to_host(&dout, &hout, st))) return rc;
    return apb_device_status(st);
}

int apb_matmul_host(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C) {
    ApiLock api_lock;
    cudaStream_t st = host_stream();
    apb_mat dA = *A, dB = *B, dC = *C;
    int rc;
    int tk = prof_begin("h2d", st);
    if ((rc = to_device(&A->b, &dA.b, 5, st, true))) return rc;
    if ((rc = to_device(&B->b, &dB.b, 10, st, true))) return rc;
    if ((rc = to_device(&C->b, &dC.b, 0, st, false))) return rc;
    prof_end(tk, st);
    if ((rc = apb_matmul(&dA, &dB, prec, algo, &dC, st))) return rc;
    tk = prof_begin("d2h", st);
    if ((rc = to_host(&dC.b, &C->b, st))) return rc;
    prof_end(tk, st);
    return apb_device_status(st);
}

// ---- pipelined matmul host entry: copy-in / compute / copy-out streams, two
// device buffer sets (workspace slots 64 + 15 k: A, B, C).  The caller's thread
// enqueues each product's copy-in and returns; a worker thread enqueues the
// product itself and its copy-out.  apb_matmul blocks its thread until the
// product's plan is read back (after the copy-in and the scan), so with the
// worker the copy-in of product i+1 is already queued behind product i's
// instead of waiting for that readback on the caller's thread.  The worker
// holds the API lock while it runs a product; every other entry point waits
// for the pipeline to empty first (ApiLock), and a device status raised by a
// pipelined product is kept for apb_matmul_host_drain.
namespace {
struct PipeJob {
    apb_mat dA, dB, dC;
    apb_balls hC;
    int64_t prec;
    int algo, k;
};
struct HostPipe {
    cudaStream_t in, comp, out;
    cudaEvent_t in_ready[2], comp_done[2], out_done[2];
    bool used[2] = {false, false};
    int next = 0;
    int err = APB_OK;
    std::string msg;
    int dev = 0;
    std::mutex mu;
    std::condition_variable cv_job, cv_done;
    std::deque<PipeJob> jobs;
    int64_t queued = 0, finished = 0;
    std::atomic<int64_t> synced{0};  // submissions known complete on the device
    HostPipe() {
        cudaGetDevice(&dev);
        cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking);
        for (int k = 0; k < 2; k++) {
            cudaEventCreateWithFlags(&in_ready[k], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&comp_done[k], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming);
        }
        std::thread([this] { run(); }).detach();  // parked on cv_job when idle; drained at exit
    }
    void record_error(int rc, const char* m) {  // caller holds mu
        if (rc && !err) {
            err = rc;
            msg = m ? m : "";
        }
    }
    // worker: product and copy-out of each submission, in submission order
    void run() {
        cudaSetDevice(dev);
        for (;;) {
            PipeJob j;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv_job.wait(lk, [&] { return !jobs.empty(); });
                j = jobs.front();
                jobs.pop_front();
            }
            int rc = APB_OK;
            std::string m;
            {
                ApiLock api_lock{ApiLock::NoDrain{}};
                cudaStreamWaitEvent(comp, in_ready[j.k], 0);
                if (used[j.k]) cudaStreamWaitEvent(comp, out_done[j.k], 0);  // set k's C has left
                if ((rc = apb_matmul(&j.dA, &j.dB, j.prec, j.algo, &j.dC, comp)) == APB_OK) {
                    cudaEventRecord(comp_done[j.k], comp);
                    cudaStreamWaitEvent(out, comp_done[j.k], 0);
                    rc = to_host(&j.dC.b, &j.hC, out);
                    cudaEventRecord(out_done[j.k], out);
                } else {
                    cudaEventRecord(comp_done[j.k], comp);
                    cudaEventRecord(out_done[j.k], out);
                }
                if (rc) m = apb_last_error();
            }
            std::lock_guard<std::mutex> lk(mu);
            used[j.k] = true;
            record_error(rc, m.c_str());
            finished++;
            cv_done.notify_all();
        }
    }
    // block until the worker has enqueued submissions [0, n)
    void wait_finished(int64_t n) {
        std::unique_lock<std::mutex> lk(mu);
        cv_done.wait(lk, [&] { return finished >= n; });
    }
    int64_t n_queued() {
        std::lock_guard<std::mutex> lk(mu);
        return queued;
    }
    // every submission enqueued and complete on the device; the device status
    // word (shared with the synchronous entries) is read under the API lock and
    // kept as the pipeline's pending error
    void settle() {
        const int64_t n = n_queued();
        wait_finished(n);
        cudaStreamSynchronize(in);
        cudaStreamSynchronize(comp);
        cudaStreamSynchronize(out);
        ApiLock api_lock{ApiLock::NoDrain{}};
        const int rc = apb_device_status(comp);
        std::lock_guard<std::mutex> lk(mu);
        record_error(rc, rc ? apb_last_error() : nullptr);
        if (synced.load() < n) synced.store(n);
    }
};
HostPipe* g_pipe = nullptr;
std::mutex g_pipe_init_mu;
HostPipe& host_pipe() {
    std::lock_guard<std::mutex> g(g_pipe_init_mu);
    if (!g_pipe) {
        g_pipe = new HostPipe;  // never destroyed: the worker thread outlives static teardown
        std::atexit([] {        // no product may still be in flight when the CUDA runtime tears down
            if (g_pipe) g_pipe->settle();
        });
    }
    return *g_pipe;
}
// would any buffer of set k have to grow (a reallocation must not race in-flight work)?
bool pipe_grows(int k, const apb_mat* A, const apb_mat* B, const apb_mat* C) {
    Workspace& ws = workspace();
    const apb_balls* bs[3] = {&A->b, &B->b, &C->b};
    for (int q = 0; q < 3; q++) {
        const size_t cnt = (size_t)bs[q]->count;
        const size_t need[5] = {cnt * bs[q]->L * 8, cnt * 8, cnt, cnt * 4, cnt * 8};
        for (int f = 0; f < 5; f++)
            if (ws.caps[64 + 15 * k + 5 * q + f] < (need[f] ? need[f] : 1)) return true;
    }
    return false;
}
}  // namespace

extern "C++" {
namespace apb {
static bool pipe_busy() { return g_pipe && g_pipe->synced.load() < g_pipe->n_queued(); }
static void pipe_quiet_drain() {
    if (g_pipe) g_pipe->settle();
}
}  // namespace apb
}

int apb_matmul_host_submit(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C) {
    HostPipe& P = host_pipe();
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != P.dev) {
        set_error("apb_matmul_host_submit: the pipeline runs on the device of its first submission");
        return APB_ERR_INVALID;
    }
    const int k = P.next;
    // submission i reuses set k of submission i-2: its product, comp_done[k] and
    // out_done[k] must be enqueued (by the worker) before they are waited on here
    P.wait_finished(P.n_queued() - 1);
    if (pipe_grows(k, A, B, C)) {  // first use / larger operands: nothing may be in flight
        P.settle();
        cudaDeviceSynchronize();
    }
    PipeJob j;
    j.dA = *A;
    j.dB = *B;
    j.dC = *C;
    j.hC = C->b;
    j.prec = prec;
    j.algo = algo;
    j.k = k;
    int rc = APB_OK;
    bool used_k;
    {
        std::lock_guard<std::mutex> lk(P.mu);
        used_k = P.used[k];
    }
    {
        // no API lock here: the copy-in touches only the pipeline's own workspace
        // slots (64..93, allocation under the workspace mutex) and its own stream,
        // so it is queued while the worker holds the lock for product i-1
        // set k's inputs were last read by the product two submissions ago
        if (used_k) cudaStreamWaitEvent(P.in, P.comp_done[k], 0);
        if (!(rc = to_device(&A->b, &j.dA.b, 64 + 15 * k, P.in, true)) &&
            !(rc = to_device(&B->b, &j.dB.b, 69 + 15 * k, P.in, true)))
            rc = to_device(&C->b, &j.dC.b, 74 + 15 * k, P.in, false);
        if (rc) {  // nothing queued: set k stays as it was; drain reports the error too
            std::lock_guard<std::mutex> lk(P.mu);
            P.record_error(rc, apb_last_error());
            return rc;
        }
        cudaEventRecord(P.in_ready[k], P.in);
    }
    P.next = k ^ 1;
    {
        std::lock_guard<std::mutex> lk(P.mu);
        P.jobs.push_back(j);
        P.queued++;
    }
    P.cv_job.notify_one();
    return APB_OK;
}

int apb_matmul_host_drain(void) {
    HostPipe& P = host_pipe();
    P.settle();
    ApiLock api_lock{ApiLock::NoDrain{}};
    int rc = cuda_check(cudaGetLastError(), "host pipeline");
    std::lock_guard<std::mutex> lk(P.mu);
    if (!rc && P.err) {
        rc = P.err;
        set_error(P.msg.c_str());
    }
    P.err = APB_OK;
    P.msg.clear();
    return rc;
}

int apb_dot_complex_batch_host(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                               const apb_balls* yim, const apb_dot_index* idx, int64_t n, int64_t batch,
                               int64_t prec, int mode, const apb_dot_tuning* tuning, apb_balls* out_re,
                               apb_balls* out_im, uint64_t* threeprod_hits) {
    ApiLock api_lock;
    cudaStream_t st = host_stream();
    apb_balls d[6] = {};
    const apb_balls* h[4] = {xre, xim, yre, yim};
    int rc;
    if (n > 0)
        for (int q = 0; q < 4; q++)  // workspace slots 32..51
            if ((rc = to_device(h[q], &d[q], 32 + 5 * q, st, true))) return rc;
    apb_balls hre = *out_re, him = *out_im;
    hre.count = him.count = batch;
    if ((rc = to_device(&hre, &d[4], 0, st, false))) return rc;
    if ((rc = to_device(&him, &d[5], 52, st, false))) return rc;
    uint64_t* dh = nullptr;
    if (threeprod_hits) {
        dh = (uint64_t*)workspace().scratch(st, 8, 57);
        if (!dh) return APB_ERR_CUDA;
        cudaMemsetAsync(dh, 0, 8, st);
    }
    if ((rc = apb_dot_complex_batch(n > 0 ? &d[0] : nullptr, n > 0 ? &d[1] : nullptr, n > 0 ? &d[2] : nullptr,
                                    n > 0 ? &d[3] : nullptr, idx, n, batch, prec, mode, tuning, &d[4], &d[5], dh,
                                    st)))
        return rc;
    if ((rc = to_host(&d[4], &hre, st))) return rc;
    if ((rc = to_host(&d[5], &him, st))) return rc;
    if (dh) cudaMemcpyAsync(threeprod_hits, dh, 8, cudaMemcpyDeviceToHost, st);
    return apb_device_status(st);
}

int apb_poly_mullow_host(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                         int64_t prec, apb_balls* out) {
    ApiLock api_lock;
    cudaStream_t st = host_stream();
    apb_balls da{}, db{}, dout{};
    int rc;
    if (alen > 0 && (rc = to_device(a, &da, 5, st, true))) return rc;
    if (blen > 0 && (rc = to_device(b, &db, 10, st, true))) return rc;
    if ((rc = to_device(out, &dout, 0, st, false))) return rc;
    if ((rc = apb_poly_mullow(alen > 0 ? &da : nullptr, alen, blen > 0 ? &db : nullptr, blen, len, prec, &dout, st)))
        return rc;
    if ((rc = to_host(&dout, out, st))) return rc;
    return apb_device_status(st);
}

int apb_series_exp_host(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out) {
    ApiLock api_lock;
    cudaStream_t st = host_stream();
    apb_balls da{}, dout{};
    int rc;
    if (alen > 0 && (rc = to_device(a, &da, 5, st, true))) return rc;
    if ((rc = to_device(out, &dout, 0, st, false))) return rc;
    if ((rc = apb_series_exp(alen > 0 ? &da : nullptr, alen, len, prec, &dout, st))) return rc;
    if ((rc = to_host(&dout, out, st))) return rc;
    return apb_device_status(st);
}

int apb_matmul_complex_host(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre,
                            const apb_mat* Bim, int64_t prec, int algo, apb_mat* Cre, apb_mat* Cim) {
    ApiLock api_lock;
    cudaStream_t st = host_stream();
    apb_mat d[6] = {*Are, *Aim, *Bre, *Bim, *Cre, *Cim};
    const apb_mat* h[6] = {Are, Aim, Bre, Bim, Cre, Cim};
    int rc;
    for (int q = 0; q < 6; q++)  // workspace slots 32..61
        if ((rc = to_device(&h[q]->b, &d[q].b, 32 + 5 * q, st, q < 4))) return rc;
    if ((rc = apb_matmul_complex(&d[0], &d[1], &d[2], &d[3], prec, algo, &d[4], &d[5], st))) return rc;
    if ((rc = to_host(&d[4].b, &Cre->b, st))) return rc;
    if ((rc = to_host(&d[5].b, &Cim->b, st))) return rc;
    return apb_device_status(st);
}

}  // extern "C"
