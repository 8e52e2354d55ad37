// pd_api.cu — implementation of the C ABI in include/pd_api.h.
//
// Validation and error codes mirror the reference's contract:
//   * N outside [1, 32]           -> PD_EINVAL  (matrix.cpp:10-15 check_qubit_count)
//   * N == 32                     -> PD_ELENGTH (matrix.cpp:17-18)
//   * n >= 4^N                    -> PD_EINVAL  (decompose.cpp:14-19 check_index)
//   * oracle with N > 6           -> PD_EINVAL  (decompose.cpp:179-181, kOracleMaxQubits)
// There is no CPU path: without an sm_100 device every compute call is PD_ENODEV.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "pd_api.h"
#include "pd_device.cuh"
#include "pd_kernels.h"
#include "pd_stage.h"


namespace {

thread_local std::string t_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    cudaGetLastError();  // clear sticky-free errors
    return fail(e == cudaErrorMemoryAllocation ? PD_ENOMEM : PD_ECUDA, "%s: %s", what,
                cudaGetErrorString(e));
}

#define PD_CUDA(call)                                       \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

constexpr unsigned kMaxQubits = 32;      // bits.hpp:15
constexpr unsigned kOracleMaxQubits = 6; // decompose.hpp:11

int check_qubits(unsigned N) {
    if (N == 0) return fail(PD_EINVAL, "a matrix needs at least one qubit (2x2)");
    if (N > kMaxQubits)
        return fail(PD_EINVAL, "qubit count %u exceeds the word-size bound of 32", N);
    if (N >= 32) return fail(PD_ELENGTH, "dense storage for 32 qubits exceeds the address space");
    return PD_OK;
}

int check_index(unsigned N, uint64_t n) {
    if (N < 32 && n >= (1ull << (2 * N)))
        return fail(PD_EINVAL, "tensor number %llu out of range for %u qubits",
                    static_cast<unsigned long long>(n), N);
    return PD_OK;
}

int check_device() {
    static std::once_flag once;
    static int status = PD_OK;
    static std::string msg;
    std::call_once(once, [] {
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            cudaGetLastError();
            status = PD_ENODEV;
            msg = std::string("no CUDA device available (") + cudaGetErrorString(e) +
                  "); this library has no CPU path";
            return;
        }
        int dev = 0, major = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        if (major != 10) {
            status = PD_ENODEV;
            msg = "device is not an sm_100 (Blackwell B200) part; kernels are built for sm_100a only";
        }
    });
    if (status != PD_OK) return fail(status, "%s", msg.c_str());
    return PD_OK;
}

uint64_t elems(unsigned N) { return 1ull << (2 * N); }

}  // namespace

struct pd_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;   // H2D, K1, even X-mask blocks
    cudaStream_t stream2 = nullptr;  // odd X-mask blocks (overlaps the previous block's tail)
    cudaStream_t d2h = nullptr;      // coefficient download, overlapped with later blocks
    cudaStream_t h2d = nullptr;      // column-segment upload, overlapped with K2 segments
    cudaStream_t gather = nullptr;   // K1 on each uploaded segment (high priority: its CTAs are
                                     // dispatched ahead of the K2 walk's pending ones)
    static constexpr int kBlocks = 48;  // >= 2^(download block bits) - 1 + tail sub-blocks
    static constexpr int kSegs = 40;    // walk segments
    cudaEvent_t gathered = nullptr;
    cudaEvent_t block_done[kBlocks] = {};
    cudaEvent_t cols_ready[kSegs] = {};
    cudaEvent_t copied[kSegs] = {};
    cudaEvent_t seg_done = nullptr;
    void* part = nullptr;            // raw partial sums between walk segments
    size_t part_bytes = 0;
    void* sel_tiles = nullptr;       // threshold selection (pd_decompose_sparse)
    size_t sel_tiles_bytes = 0;
    void* sel_idx = nullptr;
    size_t sel_idx_bytes = 0;
    void* sel_val = nullptr;
    size_t sel_val_bytes = 0;
    uint64_t sel_count = 0;
    void* g = nullptr;
    size_t g_bytes = 0;
    void* out = nullptr;
    size_t out_bytes = 0;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    void* ns = nullptr;
    size_t ns_bytes = 0;
    std::vector<pd_ctx*> subs;       // multi-device context: one sub-context per listed device
    void* stage = nullptr;           // pinned host staging (single-string diagonal)
    size_t stage_bytes = 0;
    pdb::Stager* stager = nullptr;   // pinned slot rings for pageable caller buffers (pd_stage.h)

    int ensure(void** p, size_t* have, size_t need) {
        if (*have >= need) return PD_OK;
        if (*p) cudaFree(*p);
        *p = nullptr;
        *have = 0;
        cudaError_t e = cudaMalloc(p, need);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        *have = need;
        return PD_OK;
    }
};

namespace {

// Copy to/from a host buffer; cudaMemcpyAsync handles both pinned (DMA straight
// from the caller's buffer) and pageable memory (driver-staged).
int upload(pd_ctx* ctx, void* dst, const void* src, size_t bytes) {
    PD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return PD_OK;
}

int bind(pd_ctx* ctx) {
    if (!ctx) return fail(PD_EINVAL, "null context");
    PD_CUDA(cudaSetDevice(ctx->device));
    return PD_OK;
}

// A failed host-buffer call returns only once every stream of the context (and of its
// sub-contexts) is idle: copies and kernels queued before the failure may still read the
// caller's g or write its out, and the next call would reuse ctx->g/out/part under them. The
// first error's code and message are what the caller sees.
int drained(pd_ctx* ctx, int rc) {
    if (rc == PD_OK || !ctx) return rc;
    const std::string msg = t_error;
    std::vector<pd_ctx*> all{ctx};
    all.insert(all.end(), ctx->subs.begin(), ctx->subs.end());
    for (pd_ctx* c : all) {
        if (cudaSetDevice(c->device) != cudaSuccess) continue;
        for (cudaStream_t s : {c->stream, c->stream2, c->d2h, c->h2d, c->gather})
            if (s) cudaStreamSynchronize(s);
        if (c->stager) c->stager->finish();  // host scatters into the caller's out
    }
    cudaSetDevice(ctx->device);
    cudaGetLastError();
    t_error = msg;
    return rc;
}

}  // namespace

extern "C" {

const char* pd_last_error(void) { return t_error.c_str(); }

int pd_api_version(void) { return PD_API_VERSION; }

uint64_t pd_launch_count(void) { return pdb::g_launches.load(); }

int pd_ctx_create(int device, pd_ctx** out) {
    if (!out) return fail(PD_EINVAL, "null output pointer");
    *out = nullptr;
    if (int rc = check_device()) return rc;
    int count = 0;
    PD_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
        return fail(PD_EINVAL, "device %d out of range (%d devices)", device, count);
    PD_CUDA(cudaSetDevice(device));
    pd_ctx* ctx = new pd_ctx();
    ctx->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking);
    int prio_lo = 0, prio_hi = 0;
    if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&ctx->gather, cudaStreamNonBlocking, prio_hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->gathered, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->seg_done, cudaEventDisableTiming);
    for (int b = 0; e == cudaSuccess && b < pd_ctx::kBlocks; ++b)
        e = cudaEventCreateWithFlags(&ctx->block_done[b], cudaEventDisableTiming);
    for (int b = 0; e == cudaSuccess && b < pd_ctx::kSegs; ++b)
        e = cudaEventCreateWithFlags(&ctx->cols_ready[b], cudaEventDisableTiming);
    for (int b = 0; e == cudaSuccess && b < pd_ctx::kSegs; ++b)
        e = cudaEventCreateWithFlags(&ctx->copied[b], cudaEventDisableTiming);
    if (e != cudaSuccess) {
        pd_ctx_destroy(ctx);
        return cuda_fail(e, "cudaStreamCreate");
    }
    *out = ctx;
    return PD_OK;
}

int pd_ctx_create_multi(const int* devices, int count, pd_ctx** out) {
    if (!out || !devices) return fail(PD_EINVAL, "null pointer");
    *out = nullptr;
    if (count < 1 || (count & (count - 1)) || count > 256)
        return fail(PD_EINVAL, "device count must be a power of two in [1, 256]");
    pd_ctx* parent = nullptr;
    if (int rc = pd_ctx_create(devices[0], &parent)) return rc;
    for (int k = 0; k < count; ++k) {
        pd_ctx* sub = nullptr;
        if (int rc = pd_ctx_create(devices[k], &sub)) {
            pd_ctx_destroy(parent);
            return rc;
        }
        parent->subs.push_back(sub);
    }
    *out = parent;
    return PD_OK;
}

int pd_ctx_destroy(pd_ctx* ctx) {
    if (!ctx) return PD_OK;
    for (pd_ctx* sub : ctx->subs) pd_ctx_destroy(sub);
    ctx->subs.clear();
    if (ctx->stage) cudaFreeHost(ctx->stage);
    ctx->stage = nullptr;
    cudaSetDevice(ctx->device);
    for (cudaStream_t s : {ctx->stream, ctx->stream2, ctx->d2h, ctx->h2d, ctx->gather})
        if (s) cudaStreamSynchronize(s);
    delete ctx->stager;
    ctx->stager = nullptr;
    for (void* p : {ctx->g, ctx->out, ctx->scratch, ctx->ns, ctx->part, ctx->sel_tiles, ctx->sel_idx,
                    ctx->sel_val})
        if (p) cudaFree(p);
    for (cudaEvent_t ev : {ctx->gathered, ctx->seg_done})
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : ctx->block_done)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : ctx->cols_ready)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : ctx->copied)
        if (ev) cudaEventDestroy(ev);
    for (cudaStream_t s : {ctx->stream, ctx->stream2, ctx->d2h, ctx->h2d, ctx->gather})
        if (s) cudaStreamDestroy(s);
    delete ctx;
    return PD_OK;
}

void* pd_ctx_stream(pd_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

uint64_t pd_scratch_bytes(unsigned N, uint64_t x_count, pd_path path) {
    if (N == 0 || N >= 32 || path == PD_PATH_NAIVE) return 0;
    return x_count * (1ull << N) * sizeof(double2);
}

uint64_t pd_run_offset(unsigned N, unsigned run_bits, uint64_t shard, uint64_t run) {
    // top run_bits digits: d_t = 2 z_t + (x_t ^ z_t) with x's top bits = shard, z's = run
    const unsigned low = N - run_bits;
    uint64_t top = 0;
    for (unsigned t = 0; t < run_bits; ++t) {
        const uint64_t xt = (shard >> t) & 1, zt = (run >> t) & 1;
        top |= (2 * zt + (xt ^ zt)) << (2 * t);
    }
    return top << (2 * low);
}

int pd_diag_gather_device(unsigned N, const double* g, uint64_t x0, uint64_t x_count,
                          double* diag, void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (!g || !diag) return fail(PD_EINVAL, "null buffer");
    if (int rc = check_device()) return rc;
    if (x_count == 0 || (x_count & (x_count - 1)) || x0 % x_count || x0 + x_count > (1ull << N))
        return fail(PD_EINVAL, "X-mask range must be an aligned power-of-two block inside [0, 2^N)");
    cudaError_t e = pdb::launch_diag_gather(reinterpret_cast<const double2*>(g), N, x0, x_count,
                                            reinterpret_cast<double2*>(diag),
                                            static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "diag_gather launch");
    return PD_OK;
}

int pd_copy_runs_device(const double* src, double* dst, uint64_t run_len, const uint64_t* src_off,
                        const uint64_t* dst_off, uint64_t count, void* stream) {
    if (int rc = check_device()) return rc;
    if (count && (!src || !dst || !src_off || !dst_off)) return fail(PD_EINVAL, "null buffer");
    if (count > 65535) return fail(PD_EINVAL, "at most 65535 runs per call");
    cudaError_t e = pdb::launch_copy_runs(reinterpret_cast<const double2*>(src),
                                          reinterpret_cast<double2*>(dst), run_len, src_off, dst_off,
                                          count, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "copy_runs launch");
    return PD_OK;
}

namespace {
int check_xrange(unsigned N, uint64_t x0, uint64_t x_count, unsigned run_bits, const double* out,
                 pd_layout layout) {
    if (run_bits > pdb::kMaxRunBits || run_bits > N)
        return fail(PD_EINVAL, "run_bits must be <= min(%u, N)", pdb::kMaxRunBits);
    if (x_count == 0 || (x_count & (x_count - 1)) || x0 % x_count || x0 + x_count > (1ull << N))
        return fail(PD_EINVAL, "X-mask range must be an aligned power-of-two block inside [0, 2^N)");
    if (x_count > (1ull << (N - run_bits)))
        return fail(PD_EINVAL, "X-mask range spans more than one block of 2^(N - run_bits)");
    if (layout != PD_LAYOUT_GLOBAL && layout != PD_LAYOUT_RUNS)
        return fail(PD_EINVAL, "layout must be PD_LAYOUT_GLOBAL or PD_LAYOUT_RUNS");
    if (!out) return fail(PD_EINVAL, "null output");
    return PD_OK;
}
}  // namespace

int pd_xmask_coeffs_device(unsigned N, const double* diag, uint64_t x0, uint64_t x_count,
                           unsigned run_bits, double* out, pd_layout layout, pd_path path,
                           void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = check_device()) return rc;
    if (int rc = check_xrange(N, x0, x_count, run_bits, out, layout)) return rc;
    cudaError_t e;
    const double2* d = reinterpret_cast<const double2*>(diag);
    double2* o = reinterpret_cast<double2*>(out);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (path) {
        case PD_PATH_GRAY:
            e = pdb::launch_gray_xmask(d, N, x0, x_count, run_bits, o, layout, s);
            // X-masks with an inf or NaN on their diagonal: the reference's complex products
            if (e == cudaSuccess)
                e = pdb::launch_nonfinite_fixup(d, false, N, x0, x_count,
                                                pdb::make_outmap(o, N, run_bits, layout), nullptr, s);
            break;
        case PD_PATH_WHT:
            if (N > 16) return fail(PD_EINVAL, "the WHT path supports N <= 16");
            e = pdb::launch_wht_xmask(d, N, x0, x_count, run_bits, o, layout, s);
            break;
        default: return fail(PD_EINVAL, "path must be PD_PATH_GRAY or PD_PATH_WHT");
    }
    if (e != cudaSuccess) return cuda_fail(e, "xmask coefficient launch");
    return PD_OK;
}

int pd_shard_coeffs_device(unsigned N, const double* g, uint64_t x0, uint64_t x_count,
                           unsigned run_bits, double* out, pd_layout layout, void* scratch,
                           pd_path path, void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = check_device()) return rc;
    if (!g || !scratch) return fail(PD_EINVAL, "null buffer");
    if (path == PD_PATH_WHT && pdb::wht_fused_ok(N, x_count)) {
        if (int rc = check_xrange(N, x0, x_count, run_bits, out, layout)) return rc;
        cudaError_t e = pdb::launch_wht_from_matrix(reinterpret_cast<const double2*>(g), N, x0,
                                                    x_count, static_cast<double2*>(scratch),
                                                    run_bits, reinterpret_cast<double2*>(out),
                                                    layout, static_cast<cudaStream_t>(stream));
        if (e != cudaSuccess) return cuda_fail(e, "fused WHT launch");
        return PD_OK;
    }
    if (path != PD_PATH_GRAY && path != PD_PATH_WHT)
        return fail(PD_EINVAL, "path must be PD_PATH_GRAY or PD_PATH_WHT");
    if (int rc = check_xrange(N, x0, x_count, run_bits, out, layout)) return rc;
    if (int rc = pd_diag_gather_device(N, g, x0, x_count, static_cast<double*>(scratch), stream))
        return rc;
    return pd_xmask_coeffs_device(N, static_cast<const double*>(scratch), x0, x_count, run_bits,
                                  out, layout, path, stream);
}

int pd_decompose_device(unsigned N, const double* g, double* out, void* scratch, pd_path path,
                        void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (!g || !out) return fail(PD_EINVAL, "null buffer");
    if (int rc = check_device()) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (path == PD_PATH_NAIVE) {
        cudaError_t e = pdb::launch_walk(reinterpret_cast<const double2*>(g), N, nullptr, elems(N),
                                         false, reinterpret_cast<double2*>(out), s);
        if (e != cudaSuccess) return cuda_fail(e, "walk launch");
        return PD_OK;
    }
    if (path != PD_PATH_GRAY && path != PD_PATH_WHT) return fail(PD_EINVAL, "unknown path");
    if (!scratch) return fail(PD_EINVAL, "null scratch");
    return pd_shard_coeffs_device(N, g, 0, 1ull << N, 0, out, PD_LAYOUT_GLOBAL, scratch, path,
                                  stream);
}

int pd_decompose_device_blocked(unsigned N, const double* g, double* out, void* scratch,
                                uint64_t scratch_bytes, pd_path path, void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = check_device()) return rc;
    if (path == PD_PATH_NAIVE) return pd_decompose_device(N, g, out, scratch, path, stream);
    if (path != PD_PATH_GRAY && path != PD_PATH_WHT) return fail(PD_EINVAL, "unknown path");
    if (!g || !out || !scratch) return fail(PD_EINVAL, "null buffer");
    const uint64_t dim = 1ull << N;
    uint64_t block = dim;
    while (block > 1 && pd_scratch_bytes(N, block, path) > scratch_bytes) block >>= 1;
    if (pd_scratch_bytes(N, block, path) > scratch_bytes || (block < 32 && block < dim))
        return fail(PD_EINVAL, "scratch of %llu bytes holds fewer than 32 diagonals",
                    static_cast<unsigned long long>(scratch_bytes));
    for (uint64_t x0 = 0; x0 < dim; x0 += block)
        if (int rc = pd_shard_coeffs_device(N, g, x0, block, 0, out, PD_LAYOUT_GLOBAL, scratch, path,
                                            stream))
            return rc;
    return PD_OK;
}

int pd_coeff_batch_device(unsigned N, const double* g, const uint64_t* ns, uint64_t count, int slow,
                          double* out, void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (count && (!g || !ns || !out)) return fail(PD_EINVAL, "null buffer");
    if (int rc = check_device()) return rc;
    cudaError_t e = pdb::launch_walk(reinterpret_cast<const double2*>(g), N, ns, count, slow != 0,
                                     reinterpret_cast<double2*>(out),
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "walk launch");
    return PD_OK;
}

int pd_recompose_device(unsigned N, const double* coeffs, double* g_out, void* scratch,
                        void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = check_device()) return rc;
    if (N > 16) return fail(PD_EINVAL, "recompose supports N <= 16");
    if (!coeffs || !g_out || !scratch) return fail(PD_EINVAL, "null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double2* rows = static_cast<double2*>(scratch);
    if (pdb::wht_inverse_ok(N)) {
        cudaError_t e = pdb::launch_wht_inverse(reinterpret_cast<const double2*>(coeffs), N, rows,
                                                reinterpret_cast<double2*>(g_out), s);
        if (e != cudaSuccess) return cuda_fail(e, "recompose launch");
        return PD_OK;
    }
    cudaError_t e = pdb::launch_recompose_gather(reinterpret_cast<const double2*>(coeffs), N, rows, s);
    if (e == cudaSuccess) e = pdb::launch_wht_inplace(rows, N, 1ull << N, s);
    if (e == cudaSuccess)
        e = pdb::launch_recompose_scatter(rows, N, reinterpret_cast<double2*>(g_out), s);
    if (e != cudaSuccess) return cuda_fail(e, "recompose launch");
    return PD_OK;
}

int pd_random_matrix_device(unsigned N, uint64_t seed, double* g, void* stream) {
    if (int rc = check_qubits(N)) return rc;
    if (!g) return fail(PD_EINVAL, "null buffer");
    if (int rc = check_device()) return rc;
    cudaError_t e = pdb::launch_random_matrix(N, seed, reinterpret_cast<double2*>(g),
                                              static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "random_matrix launch");
    return PD_OK;
}

// ---------------- host-buffer entry points ----------------

namespace {
int decompose_host(pd_ctx* ctx, unsigned N, const double* g, double* out, pd_path path);
}

namespace {
int decompose_multi(pd_ctx* ctx, unsigned N, const double* g, double* out, pd_path path);
}

int pd_decompose(pd_ctx* ctx, unsigned N, const double* g, double* out, pd_path path) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = bind(ctx)) return rc;
    if (!g || !out) return fail(PD_EINVAL, "null buffer");
    if (ctx->subs.size() > 1) return drained(ctx, decompose_multi(ctx, N, g, out, path));
    return drained(ctx, decompose_host(ctx, N, g, out, path));
}

namespace {
int decompose_sparse(pd_ctx* ctx, unsigned N, const double* g, pd_path path, double threshold,
                     int check_finite, uint64_t* n_kept);
}

int pd_decompose_sparse(pd_ctx* ctx, unsigned N, const double* g, pd_path path, double threshold,
                        int check_finite, uint64_t* n_kept) {
    return drained(ctx, decompose_sparse(ctx, N, g, path, threshold, check_finite, n_kept));
}

namespace {
int decompose_sparse(pd_ctx* ctx, unsigned N, const double* g, pd_path path, double threshold,
                     int check_finite, uint64_t* n_kept) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = bind(ctx)) return rc;
    if (!g || !n_kept) return fail(PD_EINVAL, "null buffer");
    if (!(threshold >= 0.0)) return fail(PD_EINVAL, "threshold must be non-negative");
    *n_kept = 0;
    if (int rc = decompose_host(ctx, N, g, nullptr, path)) return rc;  // coefficients stay on device
    const uint64_t count = elems(N);
    if (check_finite) {
        uint64_t first = 0;
        if (int rc = pd_first_nonfinite_device(static_cast<const double*>(ctx->g), count, &first,
                                               ctx->stream))
            return rc;
        if (first != UINT64_MAX)
            return fail(PD_EFORMAT, "non-finite value at row %llu, column %llu",
                        static_cast<unsigned long long>(first >> N),
                        static_cast<unsigned long long>(first & ((1ull << N) - 1)));
    }
    const uint64_t tiles = pdb::select_tiles(count);
    if (int rc = ctx->ensure(&ctx->sel_tiles, &ctx->sel_tiles_bytes,
                             tiles * sizeof(unsigned) + (tiles + 1) * sizeof(unsigned long long) + 64))
        return rc;
    if (int rc = ctx->ensure(&ctx->sel_idx, &ctx->sel_idx_bytes, count * sizeof(uint64_t))) return rc;
    if (int rc = ctx->ensure(&ctx->sel_val, &ctx->sel_val_bytes, count * sizeof(double2))) return rc;
    unsigned* tile_counts = static_cast<unsigned*>(ctx->sel_tiles);
    unsigned long long* tile_offsets = reinterpret_cast<unsigned long long*>(
        static_cast<char*>(ctx->sel_tiles) + ((tiles * sizeof(unsigned) + 63) & ~size_t{63}));
    // a slightly lowered device threshold keeps a superset; the host applies the exact
    // std::abs(c) > threshold test of io.cpp:300 to the candidates
    const double t_dev = threshold > 0.0 ? threshold * (1.0 - 1e-12) : 0.0;
    cudaError_t e = pdb::launch_select(static_cast<const double2*>(ctx->out), count, t_dev,
                                       tile_counts, tile_offsets, static_cast<uint64_t*>(ctx->sel_idx),
                                       static_cast<double2*>(ctx->sel_val), ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "select launch");
    unsigned long long kept = 0;
    PD_CUDA(cudaMemcpyAsync(&kept, tile_offsets + tiles, sizeof(kept), cudaMemcpyDeviceToHost,
                            ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->sel_count = kept;
    *n_kept = kept;
    return PD_OK;
}
}  // namespace

int pd_sparse_fetch(pd_ctx* ctx, uint64_t* idx, double* vals) {
    if (int rc = bind(ctx)) return rc;
    if (ctx->sel_count == 0) return PD_OK;
    if (!idx || !vals) return fail(PD_EINVAL, "null buffer");
    PD_CUDA(cudaMemcpyAsync(idx, ctx->sel_idx, ctx->sel_count * sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, ctx->stream));
    PD_CUDA(cudaMemcpyAsync(vals, ctx->sel_val, ctx->sel_count * sizeof(double2),
                            cudaMemcpyDeviceToHost, ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
}

int pd_first_nonfinite_device(const double* g, uint64_t count, uint64_t* first, void* stream) {
    if (int rc = check_device()) return rc;
    if (!first) return fail(PD_EINVAL, "null output");
    unsigned long long* d = nullptr;
    PD_CUDA(pdb::pool_alloc(reinterpret_cast<void**>(&d), sizeof(*d), static_cast<cudaStream_t>(stream)));
    cudaError_t e = pdb::launch_first_nonfinite(reinterpret_cast<const double2*>(g), count, d,
                                                static_cast<cudaStream_t>(stream));
    unsigned long long h = ~0ull;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
    pdb::pool_free(d, static_cast<cudaStream_t>(stream));
    if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "first_nonfinite");
    *first = h;
    return PD_OK;
}

namespace {

// Opt-in timeline of the pipelined host path (PD_E2E_TIMELINE=1): CUDA events recorded after
// each stage on the stream that ran it, printed to stderr as ms from the first upload once the
// call has synchronised (profiles/r01_e2e_timeline.txt). Off by default: no events are recorded.
struct HostTimeline {
    bool on = false;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    HostTimeline() {
        const char* e = std::getenv("PD_E2E_TIMELINE");
        on = e && e[0] == '1';
    }
    void mark(const std::string& name, cudaStream_t s) {
        if (!on) return;
        cudaEvent_t ev = nullptr;
        if (cudaEventCreate(&ev) != cudaSuccess) return;
        cudaEventRecord(ev, s);
        marks.emplace_back(name, ev);
    }
    void report() {
        if (!on || marks.empty()) return;
        for (auto& m : marks) cudaEventSynchronize(m.second);
        for (auto& m : marks) {
            float ms = 0.f;
            const cudaError_t e = cudaEventElapsedTime(&ms, marks.front().second, m.second);
            std::fprintf(stderr, "TL %-12s %9.2f%s%s\n", m.first.c_str(), ms, e ? " " : "",
                         e ? cudaGetErrorString(e) : "");
        }
    }
    ~HostTimeline() {
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
};

// the pinned slot rings of pd_stage.h, created on the first pageable call (PD_STAGE_SLOT_MB,
// PD_STAGE_WORKERS override the slot size and the worker count)
// Slots are sized to the transfer (1/16 of it, 1 – 32 MiB), so a context that only ever moves
// small matrices does not pin 640 MiB; a larger call replaces the rings once.
int stager_of(pd_ctx* ctx, size_t bytes, pdb::Stager** out, unsigned max_workers = 12) {
    const char* mb = std::getenv("PD_STAGE_SLOT_MB");
    size_t slot = mb ? static_cast<size_t>(std::max(1, std::atoi(mb))) << 20 : size_t{32} << 20;
    while (!mb && slot > (size_t{1} << 20) && slot * 16 > bytes) slot >>= 1;
    if (ctx->stager && ctx->stager->slot_bytes() < slot) {
        ctx->stager->finish();
        delete ctx->stager;
        ctx->stager = nullptr;
    }
    if (!ctx->stager) {
        const char* wk = std::getenv("PD_STAGE_WORKERS");
        const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
        const unsigned workers = wk ? static_cast<unsigned>(std::atoi(wk)) : std::min(max_workers, hw - 2);
        ctx->stager = new pdb::Stager(ctx->device, slot, 4, 16, workers);
        if (!ctx->stager->ok()) {
            delete ctx->stager;
            ctx->stager = nullptr;
            return fail(PD_ENOMEM, "cannot allocate the pinned staging slots");
        }
    }
    *out = ctx->stager;
    return PD_OK;
}

// Host <-> device copies of one host-buffer call: straight DMA for page-locked buffers, the
// pinned slot rings (pd_stage.h) for pageable ones, decided per buffer.
struct HostXfer {
    pdb::Stager* st = nullptr;
    bool up_staged = false, down_staged = false;

    // transfers below kStageMin stay with the driver's own pageable copies (a few MiB at most)
    static constexpr size_t kStageMin = size_t{8} << 20;
    int init(pd_ctx* ctx, const void* g, const void* out, size_t bytes, unsigned max_workers = 12) {
        up_staged = g && bytes >= kStageMin && pdb::host_pageable(g);
        down_staged = out && bytes >= kStageMin && pdb::host_pageable(out);
        if (up_staged || down_staged) return stager_of(ctx, bytes, &st, max_workers);
        return PD_OK;
    }
    int up2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
             cudaStream_t s) {
        const cudaError_t e = up_staged ? st->upload_2d(dst, dpitch, src, spitch, width, height, s)
                                        : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height,
                                                            cudaMemcpyHostToDevice, s);
        return e == cudaSuccess ? PD_OK : cuda_fail(e, "host upload");
    }
    int up(void* dst, const void* src, size_t bytes, cudaStream_t s) {
        return up2d(dst, bytes, src, bytes, bytes, 1, s);
    }
    // D2H once `after` (may be null) has fired
    int down(void* dst, const void* src, size_t bytes, cudaEvent_t after, cudaStream_t s) {
        cudaError_t e = cudaSuccess;
        if (down_staged) {
            e = st->download(dst, src, bytes, after, s);
        } else {
            if (after) e = cudaStreamWaitEvent(s, after, 0);
            if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
        }
        return e == cudaSuccess ? PD_OK : cuda_fail(e, "host download");
    }
    // several device -> host pieces once `after` has fired (staged: packed into shared slots)
    int down_pieces(const std::vector<pdb::Stager::Piece>& pieces, cudaEvent_t after, cudaStream_t s) {
        cudaError_t e = cudaSuccess;
        if (down_staged) {
            e = st->download(pieces.data(), pieces.size(), after, s);
        } else {
            if (after) e = cudaStreamWaitEvent(s, after, 0);
            for (size_t i = 0; e == cudaSuccess && i < pieces.size(); ++i)
                e = cudaMemcpyAsync(pieces[i].dst, pieces[i].src, pieces[i].bytes, cudaMemcpyDeviceToHost, s);
        }
        return e == cudaSuccess ? PD_OK : cuda_fail(e, "host download");
    }
    // every staged download landed in the caller's buffer
    int finish() {
        const cudaError_t e = st ? st->finish() : cudaSuccess;
        return e == cudaSuccess ? PD_OK : cuda_fail(e, "host download");
    }
};

// the host-buffer decomposition; out == nullptr leaves the coefficients in ctx->out
int decompose_host(pd_ctx* ctx, unsigned N, const double* g, double* out, pd_path path) {
    const size_t bytes = elems(N) * sizeof(double2);
    HostXfer xf;
    if (int rc = xf.init(ctx, g, out, bytes)) return rc;
    if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, bytes)) return rc;
    if (int rc = ctx->ensure(&ctx->out, &ctx->out_bytes, bytes)) return rc;
    const uint64_t sb = pd_scratch_bytes(N, 1ull << N, path);
    if (sb && ctx->scratch_bytes < sb) {
        // G and the coefficients fit but not a full set of diagonals (N = 16 on one B200:
        // 3 x 64 GiB): upload, decompose in X-mask blocks sized to what is free, download
        if (ctx->ensure(&ctx->scratch, &ctx->scratch_bytes, sb) != PD_OK) {
            size_t free_b = 0, total_b = 0;
            cudaGetLastError();
            PD_CUDA(cudaMemGetInfo(&free_b, &total_b));
            const size_t want = free_b > (1ull << 30) ? free_b - (1ull << 30) : 0;  // 1 GiB margin
            if (int rc = ctx->ensure(&ctx->scratch, &ctx->scratch_bytes, want)) return rc;
            if (int rc = xf.up(ctx->g, g, bytes, ctx->stream)) return rc;
            if (int rc = pd_decompose_device_blocked(N, static_cast<const double*>(ctx->g),
                                                     static_cast<double*>(ctx->out), ctx->scratch,
                                                     ctx->scratch_bytes, path, ctx->stream))
                return rc;
            if (out) {
                if (int rc = xf.down(out, ctx->out, bytes, nullptr, ctx->stream)) return rc;
            }
            if (int rc = xf.finish()) return rc;
            PD_CUDA(cudaStreamSynchronize(ctx->stream));
            // the scratch took all but 1 GiB of the device: give it back rather than keep it cached
            PD_CUDA(cudaFree(ctx->scratch));
            ctx->scratch = nullptr;
            ctx->scratch_bytes = 0;
            return PD_OK;
        }
    }
    const uint64_t dim = 1ull << N;
    if (path == PD_PATH_NAIVE || N < 10) {
        if (int rc = xf.up(ctx->g, g, bytes, ctx->stream)) return rc;
        if (int rc = pd_decompose_device(N, static_cast<const double*>(ctx->g),
                                         static_cast<double*>(ctx->out), ctx->scratch, path,
                                         ctx->stream))
            return rc;
        if (out) {
            if (int rc = xf.down(out, ctx->out, bytes, nullptr, ctx->stream)) return rc;
        }
        if (int rc = xf.finish()) return rc;
        PD_CUDA(cudaStreamSynchronize(ctx->stream));
        return PD_OK;
    }
    // Pipelined host path.
    //  * Upload. Gray path with >= 2 walk chunks (N >= 12): G goes up in column segments that
    //    follow the walk (chunks [1, 2), [2, 4), [4, 8) ... visit exactly the columns of the
    //    same ranges times the chunk length), each followed by K1 on those columns,
    //    while K2 runs the previous walk segment; K2 segments chain through raw partial sums,
    //    so the result is bit-identical to one launch. Otherwise G goes up in one copy.
    //  * Download. The coefficients come back in 32 X-mask blocks; block q's (32 runs of
    //    4^(N-5), pd_run_offset) are copied while later blocks compute, so only the last
    //    block's D2H is exposed; at N >= 14 the last block runs as 4 sub-blocks, so only a
    //    quarter of it is.
    double* dout = static_cast<double*>(ctx->out);
    double* diag = static_cast<double*>(ctx->scratch);
    double* gdev = static_cast<double*>(ctx->g);
    // a block's X-masks whose diagonal holds an inf or NaN get the reference's products
    // (pd_nonfinite.cu) before their download
    const pdb::OutMap gmap = pdb::make_outmap(reinterpret_cast<double2*>(dout), N, 0, PD_LAYOUT_GLOBAL);
    const bool gray = path == PD_PATH_GRAY;
    HostTimeline tl;
    // the host pipeline walks in chunks of 1024 columns (half K2's default) so that the first,
    // exposed upload is 1/16 of G at N=14
    constexpr unsigned kChunkLog = 10;  // 9 and 11 measured 500.5 and 508 ms (N=14 e2e)
    const unsigned nch = gray && pdb::gray_xmask_chunks(N) > 1 ? (1u << (N - kChunkLog)) : 1;
    const unsigned segs = nch >= pd_ctx::kSegs ? pd_ctx::kSegs : nch;
    constexpr unsigned kWhtGroupLog = 1;  // WHT host path: blocks per tile upload (log2)
    constexpr unsigned kTailLog = 2;  // last download block split in 4 (PD_E2E_TAIL)
    constexpr unsigned kBits = 5;  // 32 download blocks (N=14 e2e: 8 -> 540, 16 -> 520.4, 32 -> 518.1 ms)
    const uint64_t xc = dim >> kBits;
    const unsigned nblk = 1u << kBits;
    // the coefficients of the X-masks whose top `bits` bits equal xt: 2^bits runs of
    // 4^(N - bits), one per value of z's top bits (pd_run_offset); event slot ev
    // (block_done[ev] must have been recorded after the block's kernels)
    std::vector<pdb::Stager::Piece> pieces;
    auto download_bits = [&](unsigned bits, uint64_t xt, unsigned ev) -> int {
        if (!out) {
            PD_CUDA(cudaStreamWaitEvent(ctx->d2h, ctx->block_done[ev], 0));
            return PD_OK;
        }
        const uint64_t len = 1ull << (2 * (N - bits));
        pieces.clear();
        for (uint64_t r = 0; r < (1ull << bits); ++r) {
            const uint64_t off = 2 * pd_run_offset(N, bits, xt, r);
            pieces.push_back({out + off, dout + off, len * sizeof(double2)});
        }
        return xf.down_pieces(pieces, ctx->block_done[ev], ctx->d2h);
    };
    auto download = [&](unsigned q, cudaStream_t s) -> int {  // block q's runs, once computed
        PD_CUDA(cudaEventRecord(ctx->block_done[q], s));
        return download_bits(kBits, q, q);
    };
    // the walk segments keep raw partial sums of every coefficient (one more G-sized buffer);
    // without room for them, upload G whole and walk in one launch per download block
    bool segmented = gray && segs >= 2;
    if (segmented && ctx->ensure(&ctx->part, &ctx->part_bytes, bytes) != PD_OK) {
        cudaGetLastError();
        segmented = false;
    }
    if (segmented) {
        // Every X-mask walks the first half of the walk in segments that follow the upload; the
        // second half (with K2s the expensive one: 16 live chains per thread against <= 8) is one
        // final segment, launched per download block and alternating over two streams, so the
        // downloads overlap it. N=14 e2e 377 -> 367 ms against the PR-1 split (a quarter of the
        // X-masks segmented, the rest whole walks once G is up: with K2s the cheap early chunks
        // left the GPU idle during the upload); N=13 57.8, N=12 13.8 ms. The first-half segments
        // store raw sums and run K2q (pd_k2q.cu: 4 or 2 Z-masks per thread, so their few live
        // chains are not latency-bound while they run alone during the upload): N=14 364 -> 355.5,
        // N=13 59 -> 52.5 ms. Grouping the final blocks into launches large enough for K2s-c
        // measured no gain at N=14 (355.5) and a loss at N=13 (59.3 ms), so they stay per block.
        double2* part = static_cast<double2*>(ctx->part);
        // walk segments [bnd[k], bnd[k+1]) in chunks: `ones` single chunks (the first upload,
        // the only one not hidden behind K2, is one chunk), then aligned runs of `runlen` chunks,
        // so that the walk follows the upload instead of idling until a long segment's columns
        // have arrived (N=14 e2e, PR-1 split: doubling segments 1, 1, 2, 4, 8 510-515 ms; 4 x 1
        // then runs of 2: 500.5 ms)
        // (walking the first chunk in 2 or 4 pieces so that it starts after 1/32 or 1/64 of G:
        // 354.1 / 354.2 ms, no gain: from the third segment on the walk, not the upload, paces
        // the first half)
        constexpr unsigned ones = 4, runlen = 2;
        unsigned bnd[pd_ctx::kSegs + 1];
        unsigned nb = 0;
        bnd[nb++] = 0;
        const unsigned half = nch / 2;
        for (unsigned c = 0; c < half;) {
            unsigned L = nb - 1 < ones ? 1u : runlen;
            while (L > 1 && (c % L || c + L > half)) L >>= 1;
            if (nb == pd_ctx::kSegs) return fail(PD_EINVAL, "walk segment plan too long");
            c += L;
            bnd[nb++] = c;
        }
        bnd[nb++] = nch;
        const unsigned nseg = nb - 1;
        const uint64_t C = dim / nch;  // columns per walk chunk
        tl.mark("start", ctx->h2d);
        for (unsigned sg = 0; sg < nseg; ++sg) {
            // an aligned run of L chunks visits the aligned run of L column chunks holding gray(b)
            const uint64_t L = bnd[sg + 1] - bnd[sg];
            const uint64_t gb = bnd[sg] ^ (bnd[sg] >> 1);
            const uint64_t col0 = (gb & ~(L - 1)) * C, W = L * C;
            if (int rc = xf.up2d(gdev + 2 * col0, dim * sizeof(double2), g + 2 * col0,
                                 dim * sizeof(double2), W * sizeof(double2), dim, ctx->h2d))
                return rc;
            PD_CUDA(cudaEventRecord(ctx->copied[sg], ctx->h2d));
            tl.mark("up" + std::to_string(sg), ctx->h2d);
            PD_CUDA(cudaStreamWaitEvent(ctx->gather, ctx->copied[sg], 0));
            cudaError_t e = pdb::launch_diag_gather_cols(reinterpret_cast<const double2*>(gdev), N,
                                                         0, dim, col0, W,
                                                         reinterpret_cast<double2*>(diag), ctx->gather);
            if (e != cudaSuccess) return cuda_fail(e, "diag_gather launch");
            PD_CUDA(cudaEventRecord(ctx->cols_ready[sg], ctx->gather));
            // the walk segment over these columns is queued at once: with a pageable g the
            // next upload holds this thread while its slots fill
            if (sg + 1 < nseg) {
                PD_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->cols_ready[sg], 0));
                e = pdb::launch_gray_segment(reinterpret_cast<const double2*>(diag), N, 0, dim,
                                             bnd[sg], bnd[sg + 1], sg ? part : nullptr, part, 0,
                                             nullptr, PD_LAYOUT_GLOBAL, ctx->stream, kChunkLog);
                if (e != cudaSuccess) return cuda_fail(e, "gray segment launch");
                tl.mark("seg" + std::to_string(sg), ctx->stream);
            }
        }
        // then the final segment in download blocks (continuing from the stored raw sums) over
        // ctx->stream and stream2
        PD_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->cols_ready[nseg - 1], 0));
        PD_CUDA(cudaEventRecord(ctx->seg_done, ctx->stream));
        PD_CUDA(cudaStreamWaitEvent(ctx->stream2, ctx->seg_done, 0));
        // the last block runs as 2^tail_log sub-blocks so that only the last sub-block's
        // download is exposed after the walk ends (N=14 e2e, PD_E2E_TAIL=0/1/2/3: 355.6 / 354.6 /
        // 354.1 / 357.6 ms; smaller sub-blocks lose more to their partial last wave)
        static const char* tail_env = std::getenv("PD_E2E_TAIL");
        unsigned tail_log = tail_env ? static_cast<unsigned>(std::atoi(tail_env)) : kTailLog;
        while (tail_log && (xc >> tail_log) < 128) --tail_log;
        if (!tail_env && xc < 512) tail_log = 0;  // N=13 (256-X-mask blocks): 52.5 -> 54.0 ms split
        if (nblk - 1 + (1u << tail_log) > static_cast<unsigned>(pd_ctx::kBlocks)) tail_log = 0;
        unsigned launches = 0;
        struct Pending {
            unsigned bits;
            uint64_t xt;
            unsigned ev;
        };
        std::vector<Pending> pending;  // downloads, queued once every block is launched
        for (unsigned q = 0; q < nblk; ++q) {
            const unsigned sub_log = q + 1 == nblk ? tail_log : 0;
            const uint64_t xs = xc >> sub_log;
            for (uint64_t sb = 0; sb < (1ull << sub_log); ++sb, ++launches) {
                cudaStream_t s = (launches & 1) ? ctx->stream2 : ctx->stream;
                const uint64_t x0 = q * xc + sb * xs;
                cudaError_t e = pdb::launch_gray_segment(
                    reinterpret_cast<const double2*>(diag) + x0 * dim, N, x0, xs, bnd[nseg - 1], 0,
                    part + x0 * dim, nullptr, 0, reinterpret_cast<double2*>(dout), PD_LAYOUT_GLOBAL,
                    s, kChunkLog);
                if (e == cudaSuccess)
                    e = pdb::launch_nonfinite_fixup(reinterpret_cast<const double2*>(diag) + x0 * dim,
                                                    false, N, x0, xs, gmap, nullptr, s);
                if (e != cudaSuccess) return cuda_fail(e, "gray block launch");
                tl.mark("blk" + std::to_string(launches), s);
                PD_CUDA(cudaEventRecord(ctx->block_done[launches], s));
                pending.push_back({kBits + sub_log, (uint64_t{q} << sub_log) | sb, launches});
            }
        }
        // (a pageable out can hold this thread until a slot drains: every block is queued first)
        for (const Pending& d : pending) {
            if (int rc = download_bits(d.bits, d.xt, d.ev)) return rc;
            tl.mark("d2h" + std::to_string(d.ev), ctx->d2h);
        }
    } else {
        // WHT: block q's X-masks (top kBits bits = q) read only the tiles (t ^ q, t) of G, so G
        // goes up tile-wise per block on the copy stream and block q transforms as soon as its
        // 1/32 of G has arrived; earlier blocks' downloads overlap later blocks' uploads
        // (PCIe is full duplex), instead of the whole upload, then the whole download
        static const char* tiled_env = std::getenv("PD_E2E_WHT_TILED");
        const bool tiled = !gray && nblk <= static_cast<unsigned>(pd_ctx::kSegs) &&
                           !(tiled_env && tiled_env[0] == '0');
        static const char* grp_env = std::getenv("PD_E2E_WHT_GROUP");
        unsigned wht_grp = grp_env ? static_cast<unsigned>(std::atoi(grp_env)) : kWhtGroupLog;
        if (wht_grp > kBits) wht_grp = kBits;
        if (!tiled) {
            if (int rc = xf.up(ctx->g, g, bytes, ctx->stream)) return rc;
            if (gray && pd_diag_gather_device(N, gdev, 0, dim, diag, ctx->stream)) return PD_ECUDA;
            PD_CUDA(cudaEventRecord(ctx->gathered, ctx->stream));
            PD_CUDA(cudaStreamWaitEvent(ctx->stream2, ctx->gathered, 0));
        }
        tl.mark("start", tiled ? ctx->h2d : ctx->stream);
        for (unsigned q = 0; q < nblk; ++q) {
            cudaStream_t s = (q & 1) ? ctx->stream2 : ctx->stream;
            if (tiled) {
                // blocks go up in groups of 2^grp: for row block r the group's tiles are the
                // aligned run of 2^grp column blocks holding r ^ q, one wider copy per row block
                // (N=14 e2e, PD_E2E_WHT_GROUP=0/1/2/3, 8-64 KiB rows: 111.0 / 102.7 / 109.2 / 116.5 ms)
                const uint64_t gw = 1ull << wht_grp;
                if ((q & (gw - 1)) == 0) {
                    for (uint64_t r = 0; r < nblk; ++r) {
                        const uint64_t c0 = (r ^ q) & ~(gw - 1);
                        const uint64_t off = 2 * ((r * xc) * dim + c0 * xc);
                        if (int rc = xf.up2d(gdev + off, dim * sizeof(double2), g + off,
                                             dim * sizeof(double2), gw * xc * sizeof(double2), xc,
                                             ctx->h2d))
                            return rc;
                    }
                    PD_CUDA(cudaEventRecord(ctx->copied[q], ctx->h2d));
                    tl.mark("up" + std::to_string(q), ctx->h2d);
                }
                PD_CUDA(cudaStreamWaitEvent(s, ctx->copied[q & ~(gw - 1)], 0));
            }
            int rc;
            if (gray) {
                const double2* dq = reinterpret_cast<const double2*>(diag) + q * xc * dim;
                cudaError_t e = pdb::launch_gray_segment(dq, N, q * xc, xc, 0, 0, nullptr, nullptr, 0,
                                                         reinterpret_cast<double2*>(dout),
                                                         PD_LAYOUT_GLOBAL, s);
                if (e == cudaSuccess)
                    e = pdb::launch_nonfinite_fixup(dq, false, N, q * xc, xc, gmap, nullptr, s);
                rc = e == cudaSuccess ? PD_OK : cuda_fail(e, "gray block launch");
            } else {
                // WHT: each block gathers and transforms its own X-masks from G (fused two-pass)
                rc = pd_shard_coeffs_device(N, gdev, q * xc, xc, 0, dout, PD_LAYOUT_GLOBAL,
                                            diag + 2 * q * xc * dim, path, s);
            }
            if (rc) return rc;
            if (int rc2 = download(q, s)) return rc2;
        }
    }
    if (int rc = xf.finish()) return rc;
    PD_CUDA(cudaStreamSynchronize(ctx->d2h));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream2));
    PD_CUDA(cudaStreamSynchronize(ctx->h2d));
    PD_CUDA(cudaStreamSynchronize(ctx->gather));
    tl.report();
    return PD_OK;
}

}  // namespace

namespace {

// Multi-device host path (pd_ctx_create_multi): device g of P = 2^p owns the X-masks whose top
// p bits equal g. Its diagonals touch only the P tiles (row block t ^ g, column block t) of G,
// so it uploads exactly those (1/P of G) straight from the host, runs K1+K2 (or the WHT) on
// its block with the runs packed (PD_LAYOUT_RUNS), and downloads its 2^p runs straight to their
// offsets of the host output (in sub-blocks, overlapped with the compute of the next): every
// transfer goes over the device's own host link and there is no device-to-device traffic at
// all. The devices' work is issued asynchronously from this thread and overlaps; results are
// bit-identical to one device.
int decompose_multi(pd_ctx* ctx, unsigned N, const double* g, double* out, pd_path path) {
    const uint64_t P = ctx->subs.size();
    const unsigned p = static_cast<unsigned>(__builtin_ctzll(P));
    const uint64_t dim = 1ull << N;
    if (P > dim) return fail(PD_EINVAL, "more devices (%llu) than X-masks (%llu)",
                             static_cast<unsigned long long>(P), static_cast<unsigned long long>(dim));
    if (path != PD_PATH_GRAY && path != PD_PATH_WHT)
        return fail(PD_EINVAL, "multi-device decompositions run the GRAY or WHT path");
    const uint64_t B = dim >> p;                       // tile edge = X-masks per device
    const uint64_t run_len = 1ull << (2 * (N - p));
    // pageable host buffers go through each device's own slot rings, the workers split
    std::vector<HostXfer> xf(P);
    const unsigned q = (B >= 512) ? 2u : (B >= 256 ? 1u : 0u);
    const uint64_t Q = 1ull << q, Bs = B >> q;
    const uint64_t piece = 1ull << (2 * (N - p - q));
    for (uint64_t d = 0; d < P; ++d) {
        pd_ctx* s = ctx->subs[d];
        if (int rc = bind(s)) return rc;
        if (int rc = xf[d].init(s, g, out, (elems(N) >> p) * sizeof(double2),
                                std::max<unsigned>(2, 12 / static_cast<unsigned>(P))))
            return rc;
        const size_t gbytes = elems(N) * sizeof(double2);
        if (int rc = s->ensure(&s->g, &s->g_bytes, gbytes)) return rc;
        if (int rc = s->ensure(&s->out, &s->out_bytes, (elems(N) >> p) * sizeof(double2))) return rc;
        const uint64_t sb = pd_scratch_bytes(N, B < 32 ? 32 : B, path);
        if (int rc = s->ensure(&s->scratch, &s->scratch_bytes, sb)) return rc;
        double* gd = static_cast<double*>(s->g);
        for (uint64_t t = 0; t < P; ++t) {
            const uint64_t off = 2 * (((t ^ d) * B) * dim + t * B);  // tile (t ^ d, t), in doubles
            if (int rc = xf[d].up2d(gd + off, dim * sizeof(double2), g + off, dim * sizeof(double2),
                                    B * sizeof(double2), B, s->stream))
                return rc;
        }
        // Q sub-blocks of the device's X-masks, each downloaded while the next computes. A
        // sub-block writes into the device's packed runs (rb = p, the fast run-pointer K2); its
        // coefficients there are P Q contiguous pieces of 4^(N-p-q): z's top p bits r select the
        // run, the next q digits (from x bits s and z bits u) the piece.
        double* so = static_cast<double*>(s->out);
        for (uint64_t sb_i = 0; sb_i < Q; ++sb_i) {
            if (int rc = pd_shard_coeffs_device(N, gd, d * B + sb_i * Bs, Bs, p, so, PD_LAYOUT_RUNS,
                                                s->scratch, path, s->stream))
                return rc;
            PD_CUDA(cudaEventRecord(s->block_done[sb_i], s->stream));
        }
    }
    // every device's work is queued before any download: a pageable out can hold this thread
    // until a staging slot drains
    std::vector<pdb::Stager::Piece> pieces;
    for (uint64_t d = 0; d < P; ++d) {
        pd_ctx* s = ctx->subs[d];
        if (int rc = bind(s)) return rc;
        double* so = static_cast<double*>(s->out);
        for (uint64_t sb_i = 0; sb_i < Q; ++sb_i) {
            pieces.clear();
            for (uint64_t r = 0; r < P; ++r)
                for (uint64_t u = 0; u < Q; ++u) {
                    const uint64_t host_off = pd_run_offset(N, p + q, d * Q + sb_i, r * Q + u);
                    const uint64_t dev_off = r * run_len + (pd_run_offset(q, q, sb_i, u) << (2 * (N - p - q)));
                    pieces.push_back({out + 2 * host_off, so + 2 * dev_off, piece * sizeof(double2)});
                }
            if (int rc = xf[d].down_pieces(pieces, s->block_done[sb_i], s->d2h)) return rc;
        }
    }
    for (uint64_t d = 0; d < P; ++d) {
        pd_ctx* s = ctx->subs[d];
        if (int rc = bind(s)) return rc;
        if (int rc = xf[d].finish()) return rc;
        PD_CUDA(cudaStreamSynchronize(s->d2h));
        PD_CUDA(cudaStreamSynchronize(s->stream));
    }
    return bind(ctx);
}

}  // namespace

int pd_random_matrix(pd_ctx* ctx, unsigned N, uint64_t seed, double* g_out) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = bind(ctx)) return rc;
    if (!g_out) return fail(PD_EINVAL, "null buffer");
    const size_t bytes = elems(N) * sizeof(double2);
    if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, bytes)) return rc;
    if (int rc = pd_random_matrix_device(N, seed, static_cast<double*>(ctx->g), ctx->stream)) return rc;
    HostXfer xf;  // to host memory of either kind (pageable: the staging slots)
    int rc = xf.init(ctx, nullptr, g_out, bytes);
    if (rc == PD_OK) rc = xf.down(g_out, ctx->g, bytes, nullptr, ctx->stream);
    if (rc == PD_OK) rc = xf.finish();
    if (rc != PD_OK) return drained(ctx, rc);
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
}

namespace {
// host buffers of either kind (HostXfer: pinned by DMA, pageable through the staging slots)
int recompose_host(pd_ctx* ctx, unsigned N, const double* coeffs, double* g_out) {
    const size_t bytes = elems(N) * sizeof(double2);
    if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, bytes)) return rc;
    if (int rc = ctx->ensure(&ctx->out, &ctx->out_bytes, bytes)) return rc;
    if (int rc = ctx->ensure(&ctx->scratch, &ctx->scratch_bytes, bytes)) return rc;
    HostXfer xf;
    if (int rc = xf.init(ctx, coeffs, g_out, bytes)) return rc;
    if (int rc = xf.up(ctx->out, coeffs, bytes, ctx->stream)) return rc;
    if (int rc = pd_recompose_device(N, static_cast<const double*>(ctx->out),
                                     static_cast<double*>(ctx->g), ctx->scratch, ctx->stream))
        return rc;
    if (int rc = xf.down(g_out, ctx->g, bytes, nullptr, ctx->stream)) return rc;
    if (int rc = xf.finish()) return rc;
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
}
}  // namespace

int pd_recompose(pd_ctx* ctx, unsigned N, const double* coeffs, double* g_out) {
    if (int rc = check_qubits(N)) return rc;
    if (int rc = bind(ctx)) return rc;
    if (!coeffs || !g_out) return fail(PD_EINVAL, "null buffer");
    return drained(ctx, recompose_host(ctx, N, coeffs, g_out));
}

namespace {
int coeff_batch_host(pd_ctx* ctx, unsigned N, const double* g, const uint64_t* ns, uint64_t count,
                     double* out);
}

int pd_coeff_batch(pd_ctx* ctx, unsigned N, const double* g, const uint64_t* ns, uint64_t count,
                   double* out) {
    if (int rc = check_qubits(N)) return rc;
    if (count && (!g || !ns || !out)) return fail(PD_EINVAL, "null buffer");
    for (uint64_t k = 0; k < count; ++k)
        if (int rc = check_index(N, ns[k])) return rc;
    if (int rc = bind(ctx)) return rc;
    if (count == 0) return PD_OK;
    return drained(ctx, coeff_batch_host(ctx, N, g, ns, count, out));
}

namespace {
int coeff_batch_host(pd_ctx* ctx, unsigned N, const double* g, const uint64_t* ns, uint64_t count,
                     double* out) {
    const size_t gbytes = elems(N) * sizeof(double2);
    const uint64_t dim = 1ull << N;
    // few X-masks among the strings (at most 2^N / 8): upload only their gathered diagonals
    std::vector<uint64_t> xs(count);
    for (uint64_t k = 0; k < count; ++k) xs[k] = pdb::xmask_of(ns[k]);
    std::vector<uint64_t> uniq(xs);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    if (N >= 4 && uniq.size() * 8 <= dim) {
        const uint64_t m = uniq.size();
        const size_t dbytes = m * dim * sizeof(double2);
        const size_t need = dbytes + count * (sizeof(uint64_t) + sizeof(uint32_t));
        if (ctx->stage_bytes < need) {
            if (ctx->stage) cudaFreeHost(ctx->stage);
            ctx->stage = nullptr;
            ctx->stage_bytes = 0;
            PD_CUDA(cudaHostAlloc(&ctx->stage, need, cudaHostAllocDefault));
            ctx->stage_bytes = need;
        }
        double* d = static_cast<double*>(ctx->stage);
        for (uint64_t j = 0; j < m; ++j)
            for (uint64_t i = 0; i < dim; ++i) {
                const double* e = g + 2 * ((i ^ uniq[j]) * dim + i);
                d[2 * (j * dim + i)] = e[0];
                d[2 * (j * dim + i) + 1] = e[1];
            }
        uint64_t* nsh = reinterpret_cast<uint64_t*>(static_cast<char*>(ctx->stage) + dbytes);
        uint32_t* slot = reinterpret_cast<uint32_t*>(nsh + count);
        std::memcpy(nsh, ns, count * sizeof(uint64_t));
        for (uint64_t k = 0; k < count; ++k)
            slot[k] = static_cast<uint32_t>(std::lower_bound(uniq.begin(), uniq.end(), xs[k]) - uniq.begin());
        if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, need)) return rc;
        if (int rc = ctx->ensure(&ctx->out, &ctx->out_bytes, count * sizeof(double2))) return rc;
        PD_CUDA(cudaMemcpyAsync(ctx->g, ctx->stage, need, cudaMemcpyHostToDevice, ctx->stream));
        const char* base = static_cast<const char*>(ctx->g);
        cudaError_t e = pdb::launch_walk_slots(
            reinterpret_cast<const double2*>(base), N, reinterpret_cast<const uint64_t*>(base + dbytes),
            reinterpret_cast<const uint32_t*>(base + dbytes + count * sizeof(uint64_t)), count,
            static_cast<double2*>(ctx->out), ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "walk launch");
        PD_CUDA(cudaMemcpyAsync(out, ctx->out, count * sizeof(double2), cudaMemcpyDeviceToHost,
                                ctx->stream));
        PD_CUDA(cudaStreamSynchronize(ctx->stream));
        return PD_OK;
    }
    if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, gbytes)) return rc;
    if (int rc = ctx->ensure(&ctx->ns, &ctx->ns_bytes, count * sizeof(uint64_t))) return rc;
    if (int rc = ctx->ensure(&ctx->out, &ctx->out_bytes, count * sizeof(double2))) return rc;
    HostXfer xf;  // the matrix from host memory of either kind (pageable: the staging slots)
    if (int rc = xf.init(ctx, g, nullptr, gbytes)) return rc;
    if (int rc = xf.up(ctx->g, g, gbytes, ctx->stream)) return rc;
    if (int rc = upload(ctx, ctx->ns, ns, count * sizeof(uint64_t))) return rc;
    if (int rc = pd_coeff_batch_device(N, static_cast<const double*>(ctx->g),
                                       static_cast<const uint64_t*>(ctx->ns), count, 0,
                                       static_cast<double*>(ctx->out), ctx->stream))
        return rc;
    PD_CUDA(cudaMemcpyAsync(out, ctx->out, count * sizeof(double2), cudaMemcpyDeviceToHost,
                            ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
}
}  // namespace

int pd_coeff(pd_ctx* ctx, unsigned N, const double* g, uint64_t n, int slow, double* out) {
    if (int rc = check_qubits(N)) return rc;
    if (!g || !out) return fail(PD_EINVAL, "null buffer");
    if (int rc = check_index(N, n)) return rc;
    if (int rc = bind(ctx)) return rc;
    // one string reads one XOR-diagonal: gather its 2^N elements on the host (16 KiB at N=10,
    // 256 KiB at N=14) instead of uploading the whole matrix, then walk it in the reference's
    // order on the device (K3 over the compact diagonal; bit-identical to the full-matrix walk)
    const uint64_t dim = 1ull << N;
    const uint64_t x = pdb::xmask_of(n);
    const size_t dbytes = dim * sizeof(double2) + sizeof(uint64_t);
    if (ctx->stage_bytes < dbytes) {
        if (ctx->stage) cudaFreeHost(ctx->stage);
        ctx->stage = nullptr;
        ctx->stage_bytes = 0;
        PD_CUDA(cudaHostAlloc(&ctx->stage, dbytes, cudaHostAllocDefault));
        ctx->stage_bytes = dbytes;
    }
    double* d = static_cast<double*>(ctx->stage);
    for (uint64_t i = 0; i < dim; ++i) {
        const double* e = g + 2 * ((i ^ x) * dim + i);
        d[2 * i] = e[0];
        d[2 * i + 1] = e[1];
    }
    std::memcpy(d + 2 * dim, &n, sizeof(n));
    if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, dbytes)) return rc;
    if (int rc = ctx->ensure(&ctx->out, &ctx->out_bytes, sizeof(double2))) return rc;
    PD_CUDA(cudaMemcpyAsync(ctx->g, d, dbytes, cudaMemcpyHostToDevice, ctx->stream));
    const double2* dd = static_cast<const double2*>(ctx->g);
    cudaError_t e = pdb::launch_walk_diag(dd, N, reinterpret_cast<const uint64_t*>(dd + dim), slow != 0,
                                          static_cast<double2*>(ctx->out), ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "walk launch");
    PD_CUDA(cudaMemcpyAsync(out, ctx->out, sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
}

int pd_oracle_coeff(pd_ctx* ctx, unsigned N, const double* g, uint64_t n, double* out) {
    if (int rc = check_qubits(N)) return rc;
    if (!g || !out) return fail(PD_EINVAL, "null buffer");
    if (int rc = check_index(N, n)) return rc;
    if (N > kOracleMaxQubits)
        return fail(PD_EINVAL, "reference path is capped at %u qubits", kOracleMaxQubits);
    if (int rc = bind(ctx)) return rc;
    const size_t gbytes = elems(N) * sizeof(double2);
    if (int rc = ctx->ensure(&ctx->g, &ctx->g_bytes, gbytes)) return rc;
    if (int rc = ctx->ensure(&ctx->out, &ctx->out_bytes, sizeof(double2))) return rc;
    if (int rc = upload(ctx, ctx->g, g, gbytes)) return rc;
    cudaError_t e = pdb::launch_kron_trace(static_cast<const double2*>(ctx->g), N, n,
                                           static_cast<double2*>(ctx->out), ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "kron_trace launch");
    PD_CUDA(cudaMemcpyAsync(out, ctx->out, sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
    PD_CUDA(cudaStreamSynchronize(ctx->stream));
    return PD_OK;
}

namespace {
typedef int (*MemGetAddressRange)(unsigned long long*, size_t*, unsigned long long);

int allocation_base(const void* p, uintptr_t* base) {
    static MemGetAddressRange fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<MemGetAddressRange>(f);
    }();
    if (!fn) return fail(PD_ECUDA, "cuMemGetAddressRange unavailable");
    unsigned long long b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0)
        return fail(PD_EINVAL, "pointer %p is not device memory", p);
    *base = static_cast<uintptr_t>(b);
    return PD_OK;
}

std::mutex g_ipc_mu;
std::vector<std::pair<void*, void*>> g_ipc_open;  // (returned pointer, mapped base)
}  // namespace

int pd_ipc_export(const void* dev_ptr, pd_ipc_handle* out) {
    if (int rc = check_device()) return rc;
    if (!dev_ptr || !out) return fail(PD_EINVAL, "null pointer");
    uintptr_t base = 0;
    if (int rc = allocation_base(dev_ptr, &base)) return rc;
    cudaIpcMemHandle_t h;
    PD_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) <= sizeof(out->bytes), "IPC handle size");
    std::memset(out->bytes, 0, sizeof(out->bytes));
    std::memcpy(out->bytes, &h, sizeof(h));
    out->offset = reinterpret_cast<uintptr_t>(dev_ptr) - base;
    return PD_OK;
}

int pd_ipc_open(const pd_ipc_handle* handle, void** dev_ptr) {
    if (int rc = check_device()) return rc;
    if (!handle || !dev_ptr) return fail(PD_EINVAL, "null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle->bytes, sizeof(h));
    void* base = nullptr;
    PD_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = static_cast<char*>(base) + handle->offset;
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    g_ipc_open.emplace_back(*dev_ptr, base);
    return PD_OK;
}

int pd_ipc_close(void* dev_ptr) {
    void* base = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_ipc_mu);
        for (size_t i = 0; i < g_ipc_open.size(); ++i)
            if (g_ipc_open[i].first == dev_ptr) {
                base = g_ipc_open[i].second;
                g_ipc_open.erase(g_ipc_open.begin() + static_cast<long>(i));
                break;
            }
    }
    if (!base) return fail(PD_EINVAL, "pointer %p was not opened by pd_ipc_open", dev_ptr);
    PD_CUDA(cudaIpcCloseMemHandle(base));
    return PD_OK;
}

int pd_host_alloc(size_t bytes, void** out) {
    if (!out) return fail(PD_EINVAL, "null output pointer");
    *out = nullptr;
    if (int rc = check_device()) return rc;
    PD_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
    return PD_OK;
}

int pd_host_free(void* p) {
    if (p) PD_CUDA(cudaFreeHost(p));
    return PD_OK;
}

int pd_fp64_add_probe(pd_ctx* ctx, double* dadd_per_s) {
    if (int rc = bind(ctx)) return rc;
    if (!dadd_per_s) return fail(PD_EINVAL, "null output");
    int sms = 0;
    PD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    double* sink = nullptr;
    PD_CUDA(cudaMalloc(&sink, sizeof(double)));
    const unsigned blocks = static_cast<unsigned>(sms) * 8, iters = 1u << 15;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaError_t e = pdb::launch_fp64_probe(blocks, iters, sink, ctx->stream);  // warm-up
    float ms = 0.f;
    if (e == cudaSuccess) {
        cudaEventRecord(a, ctx->stream);
        e = pdb::launch_fp64_probe(blocks, iters, sink, ctx->stream);
        cudaEventRecord(b, ctx->stream);
        if (e == cudaSuccess) e = cudaEventSynchronize(b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return cuda_fail(e, "fp64 probe");
    const double dadds = static_cast<double>(blocks) * 256.0 * 16.0 * iters;
    *dadd_per_s = dadds / (ms * 1e-3);
    return PD_OK;
}

}  // extern "C"
