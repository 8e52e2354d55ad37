/*
 * pd_api.h — C ABI of the B200 Pauli-decomposition library (libpd_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (arXiv 2401.16378, proj/) has no FFI of its own: its boundary is the C++
 * declarations in proj/include/paulidecomp/decompose.hpp:33-56 and
 * matrix.hpp:14-51, exposed to Python by proj/bindings/module.cpp:56-121.
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions (all functions):
 *   - plain pointers and sizes; no C++ or CUDA types. Matrices are row-major
 *     dim x dim complex128 stored as interleaved (re, im) doubles — the layout
 *     of std::complex<double> / numpy complex128 — so element (row j, col i)
 *     is at doubles [2*(j*dim+i), 2*(j*dim+i)+1] (matrix.hpp:10-13).
 *   - coefficient arrays are indexed by tensor number n: base-4 digit t of n
 *     selects sigma_t in {I,X,Y,Z}, digit 0 rightmost (pauli.hpp:13-20).
 *   - return value is a pd_status; on failure pd_last_error() holds the message
 *     (thread-local). PD_EINVAL / PD_ELENGTH mirror std::invalid_argument /
 *     std::length_error thrown by the reference (decompose.cpp:14-19,98-99;
 *     matrix.cpp:10-19).
 *   - *_device functions take device pointers and a cudaStream_t passed as
 *     void* (NULL = legacy default stream) and are stream-ordered; host-buffer
 *     functions are synchronous, like the reference's calls.
 *   - there is no CPU fallback: without a usable sm_100 GPU every compute
 *     entry point returns PD_ENODEV.
 */
#ifndef PD_API_H
#define PD_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PD_API_VERSION 3

#if defined(__GNUC__)
#define PD_EXPORT __attribute__((visibility("default")))
#else
#define PD_EXPORT
#endif

typedef enum pd_status {
    PD_OK = 0,
    PD_EINVAL = -1,  /* std::invalid_argument in the reference */
    PD_ELENGTH = -2, /* std::length_error */
    PD_ENOMEM = -3,  /* std::bad_alloc / cudaErrorMemoryAllocation */
    PD_ECUDA = -4,   /* any other CUDA runtime failure */
    PD_ENODEV = -5,  /* no CUDA device, or not an sm_100 part */
    PD_EFORMAT = -6  /* malformed data, e.g. a non-finite matrix element (FormatError) */
} pd_status;

typedef enum pd_path {
    PD_PATH_GRAY = 0,  /* K1 diagonal gather + K2 Gray-code FP64 sum (the paper's O(8^N) method) */
    PD_PATH_WHT = 1,   /* K1 + fast Walsh-Hadamard butterflies (separately reported second path) */
    PD_PATH_NAIVE = 2  /* K0: one thread per n, reference-order walk straight from G */
} pd_path;

/* Where the coefficients of an X-mask range go (pd_xmask_coeffs_device, pd_shard_coeffs_device). */
typedef enum pd_layout {
    PD_LAYOUT_GLOBAL = 0, /* out[n]: the reference-ordered array of all 4^N coefficients */
    PD_LAYOUT_RUNS = 1    /* out is the range's block of 4^N / 2^run_bits coefficients, packed
                             as its 2^run_bits runs (see pd_xmask_coeffs_device) */
} pd_layout;

typedef struct pd_ctx pd_ctx;

PD_EXPORT const char* pd_last_error(void);
PD_EXPORT int pd_api_version(void);

/* Device context: binds a CUDA device and owns a stream plus cached scratch.
 * One host thread per context (the reference's calls are synchronous). */
PD_EXPORT int pd_ctx_create(int device, pd_ctx** out);
PD_EXPORT int pd_ctx_destroy(pd_ctx* ctx);
/* Multi-device context over count = 2^p GPUs of one host (a device may be listed more than
 * once). pd_decompose on it splits the X-masks across the devices: device g uploads only the
 * 1/P of G its diagonals touch, computes its block and downloads its coefficient runs straight
 * into `out`, with no device-to-device traffic; results are bit-identical to one device. The
 * multi-device analogue of decompose_parallel's `threads` (decompose.cpp:95-131). */
PD_EXPORT int pd_ctx_create_multi(const int* devices, int count, pd_ctx** out);
/* the context's stream, as a cudaStream_t */
PD_EXPORT void* pd_ctx_stream(pd_ctx* ctx);

/* ---------------- host-buffer entry points (synchronous) ---------------- */

/* All 4^N coefficients of the 2^N x 2^N matrix g, written to out (2*4^N doubles).
 * Replaces decompose_parallel(const DenseMatrix&, unsigned threads)
 * (decompose.hpp:46, decompose.cpp:95-131,205-207) and
 * decompose_serial_quaternary (decompose.hpp:55; same output).
 * g and out may be page-locked (cudaHostAlloc / cudaHostRegister: copied by DMA directly) or
 * ordinary pageable memory (copied through the context's pinned staging slots on host worker
 * threads; env PD_STAGE_WORKERS, PD_STAGE_SLOT_MB), decided per buffer. On any error the call
 * returns only after all of its queued copies and kernels have finished, so the caller may
 * free g and out at once. */
PD_EXPORT int pd_decompose(pd_ctx* ctx, unsigned num_qubits, const double* g, double* out, pd_path path);

/* One coefficient c_n, written to out[0..1].
 * Replaces coeff_fast(const DenseMatrix&, uint64_t n) (decompose.hpp:33,
 * decompose.cpp:49-57,156-159); slow != 0 replaces coeff_slow (decompose.hpp:35). */
PD_EXPORT int pd_coeff(pd_ctx* ctx, unsigned num_qubits, const double* g, uint64_t n, int slow, double* out);

/* Many coefficients of one matrix: out[2k..2k+1] = c_{ns[k]}. Batched form of
 * coeff_fast (decompose.hpp:33), one call instead of `count` calls. */
PD_EXPORT int pd_coeff_batch(pd_ctx* ctx, unsigned num_qubits, const double* g, const uint64_t* ns,
                   uint64_t count, double* out);

/* Brute-force Kronecker-product trace Tr(P_n G)/2^N, N <= 6.
 * Replaces oracle_coeff_kron (decompose.hpp:37, decompose.cpp:176-203). */
PD_EXPORT int pd_oracle_coeff(pd_ctx* ctx, unsigned num_qubits, const double* g, uint64_t n, double* out);

/* Dense matrix sum_n c_n P_n from all 4^N coefficients (2*4^N doubles) into g_out
 * (2*4^N doubles). Replaces recompose(const PauliDecomposition&) (decompose.hpp:59,
 * decompose.cpp:221-250). N <= 16. */
PD_EXPORT int pd_recompose(pd_ctx* ctx, unsigned num_qubits, const double* coeffs, double* g_out);

/* Decompose g and keep on the device only the coefficients with |c_n| > threshold (all when
 * threshold == 0), in ascending tensor-number order: the selection of the reference's CSV
 * writer (io.cpp:286-307) done before any D2H. *n_kept receives the count; pd_sparse_fetch
 * copies the kept tensor numbers and coefficients out. The device selection is a superset
 * within 1e-12 relative of the threshold; apply |c| > threshold exactly on the host.
 * check_finite != 0 rejects non-finite elements with PD_EFORMAT (the readers' rule,
 * io.cpp:118-123), checked on the device copy of g. */
PD_EXPORT int pd_decompose_sparse(pd_ctx* ctx, unsigned num_qubits, const double* g, pd_path path,
                                  double threshold, int check_finite, uint64_t* n_kept);
PD_EXPORT int pd_sparse_fetch(pd_ctx* ctx, uint64_t* idx, double* vals);

/* ---------------- device-resident entry points (stream-ordered) ---------------- */

/* Scratch bytes pd_decompose_device needs for `path` (0 for PD_PATH_NAIVE). */
PD_EXPORT uint64_t pd_scratch_bytes(unsigned num_qubits, uint64_t x_count, pd_path path);

/* Full decomposition of a device-resident matrix into a device coefficient array,
 * using caller-provided scratch (>= pd_scratch_bytes(N, 2^N, path)). */
PD_EXPORT int pd_decompose_device(unsigned num_qubits, const double* g, double* out, void* scratch,
                        pd_path path, void* stream);

/* pd_decompose_device with a scratch buffer of any size >= pd_scratch_bytes(N, 32, path): the
 * X-masks are processed in the largest power-of-two blocks whose diagonals fit scratch_bytes.
 * This is what lets one 180 GB B200 hold N = 16 (G and the coefficients, 64 GiB each, plus a
 * block of diagonals) where the one-shot form would need 192 GiB. */
PD_EXPORT int pd_decompose_device_blocked(unsigned num_qubits, const double* g, double* out,
                                          void* scratch, uint64_t scratch_bytes, pd_path path,
                                          void* stream);

/* K1: diag[(x - x0) * dim + i] = G[i ^ x][i] for x in [x0, x0 + x_count).
 * x_count is a power of two and x0 a multiple of it. */
PD_EXPORT int pd_diag_gather_device(unsigned num_qubits, const double* g, uint64_t x0, uint64_t x_count,
                          double* diag, void* stream);

/* K2 (path GRAY) or K4 (path WHT): every coefficient whose X-mask lies in
 * [x0, x0 + x_count), from the gathered diagonals. Output addressing follows the
 * X-mask sharding of the multi-GPU layer: with run_bits = p, the X-masks whose top p
 * bits equal g (block g of 2^p) own 2^p contiguous runs of 4^(N-p) coefficients of the
 * reference-ordered array, one per value r of the top p bits of the Z-mask, starting at
 * pd_run_offset(N, p, g, r). The range must lie inside one such block.
 *   PD_LAYOUT_GLOBAL: coefficient n goes to out[n] (out holds all 4^N; p is irrelevant).
 *   PD_LAYOUT_RUNS:   out holds the block's runs back to back: run r at out + r 4^(N-p),
 *                     so a block (a GPU's shard, or one pipelined sub-block) is contiguous.
 * p <= min(N, 8). out is 2 doubles per coefficient. */
PD_EXPORT int pd_xmask_coeffs_device(unsigned num_qubits, const double* diag, uint64_t x0, uint64_t x_count,
                           unsigned run_bits, double* out, pd_layout layout, pd_path path, void* stream);

/* Every coefficient whose X-mask lies in [x0, x0 + x_count), straight from the matrix g,
 * with the output addressing of pd_xmask_coeffs_device. GRAY: K1 into scratch, then K2.
 * WHT: the fused two-pass transform (pass 1 gathers and butterflies the low 7 index bits
 * into scratch, pass 2 the high bits) when N in [8,16] and x_count >= 32, else K1 + K4.
 * scratch >= pd_scratch_bytes(N, x_count, path). This is one X-mask shard's work. */
PD_EXPORT int pd_shard_coeffs_device(unsigned num_qubits, const double* g, uint64_t x0,
                                     uint64_t x_count, unsigned run_bits, double* out,
                                     pd_layout layout, void* scratch, pd_path path, void* stream);

/* Global offset (in coefficients) of run r of X-mask shard g for p = run_bits. */
PD_EXPORT uint64_t pd_run_offset(unsigned num_qubits, unsigned run_bits, uint64_t shard, uint64_t run);

/* Device form of pd_recompose; scratch >= 16 * 4^N bytes. */
PD_EXPORT int pd_recompose_device(unsigned num_qubits, const double* coeffs, double* g_out, void* scratch,
                        void* stream);

/* K3: out[k] = c_{ns[k]} for a device list of tensor numbers (reference-order walk). */
PD_EXPORT int pd_coeff_batch_device(unsigned num_qubits, const double* g, const uint64_t* ns, uint64_t count,
                          int slow, double* out, void* stream);

/* random_matrix(N, seed) (bench.cpp:48-58) generated on the device and copied to g_out
 * (2*4^N doubles); bit-identical to the reference's host generator. */
PD_EXPORT int pd_random_matrix(pd_ctx* ctx, unsigned num_qubits, uint64_t seed, double* g_out);

/* Device restatement of the reference's seeded generator random_matrix(N, seed)
 * (bench.cpp:16-58); bit-identical to it. */
PD_EXPORT int pd_random_matrix_device(unsigned num_qubits, uint64_t seed, double* g, void* stream);

/* Index of the first complex element of g[0..count) with a non-finite part, or UINT64_MAX;
 * synchronous on `stream`. */
PD_EXPORT int pd_first_nonfinite_device(const double* g, uint64_t count, uint64_t* first,
                                        void* stream);

/* Page-locked host memory for the host-buffer entry points (H2D/D2H at full PCIe rate). */
PD_EXPORT int pd_host_alloc(size_t bytes, void** out);
PD_EXPORT int pd_host_free(void* p);

/* ---------------- NCCL pipeline pieces (multi-GPU sharding, sharding.py) ----------------
 * The pipelined NCCL mode splits each rank's X-masks into blocks: rank 0 gathers block j's
 * diagonals of every rank (pd_diag_gather_device, row-major: one contiguous message per rank),
 * every rank walks block j as soon as its rows are in (pd_xmask_coeffs_device), and each
 * finished block's 2^(p+q) coefficient runs go back to rank 0 as one message while the next
 * block computes. The reference's own parallel split is decompose.cpp:95-131. */

/* dst[dst_off[k] + j] = src[src_off[k] + j] for j < run_len, k < count: packing / unpacking
 * coefficient runs (offset tables are device arrays of element offsets, count <= 65535). */
PD_EXPORT int pd_copy_runs_device(const double* src, double* dst, uint64_t run_len,
                                  const uint64_t* src_off, const uint64_t* dst_off, uint64_t count,
                                  void* stream);

/* ---------------- peer memory (multi-GPU sharding over NVLink) ---------------- */

/* A device buffer exported to the other processes of one box: the CUDA IPC handle of the
 * allocation that contains it plus the buffer's offset inside that allocation (so buffers
 * sub-allocated by a caching allocator can be shared). Plain bytes: send it through any
 * host channel (the sharding layer uses torch.distributed object collectives). */
typedef struct pd_ipc_handle {
    unsigned char bytes[64];
    uint64_t offset;
} pd_ipc_handle;

/* Export the allocation containing dev_ptr. */
PD_EXPORT int pd_ipc_export(const void* dev_ptr, pd_ipc_handle* out);
/* Map a peer's exported buffer into this process on the current device (peer access over
 * NVLink/NVSwitch when the owner is another GPU); *dev_ptr = mapped base + offset. The kernels
 * take such pointers like local ones: K1 gathers diagonals straight from the owner's G and K2
 * stores coefficients straight into the owner's output (pd_shard_coeffs_device with
 * PD_LAYOUT_GLOBAL), which replaces the broadcast and the gather of the NCCL sharding mode. */
PD_EXPORT int pd_ipc_open(const pd_ipc_handle* handle, void** dev_ptr);
/* Unmap a pointer returned by pd_ipc_open. */
PD_EXPORT int pd_ipc_close(void* dev_ptr);

/* ---------------- measurement helpers ---------------- */

/* Number of kernels this library has launched in this process (all threads). */
PD_EXPORT uint64_t pd_launch_count(void);

/* FP64-add issue probe: runs a pure-DADD kernel over all SMs on the context's
 * device and returns the achieved DADD/s in *dadd_per_s. */
PD_EXPORT int pd_fp64_add_probe(pd_ctx* ctx, double* dadd_per_s);

#ifdef __cplusplus
}
#endif

#endif /* PD_API_H */
