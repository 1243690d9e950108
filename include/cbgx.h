/*
 * cbgx.h -- C-ABI of the B200-native FRSZ2 / compressed-basis GMRES path.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/cbg/{frsz2,basis,sparse,gmres}.hpp). Plain C
 * types, caller-owned buffers, no exceptions across the boundary:
 * every entry point returns a status (CBGX_OK = 0) and cbgx_last_error()
 * gives the message of the calling thread's last failure. The C++ wrappers in
 * include/cbg/*.hpp (libcbg_b200.so) turn statuses back into the
 * reference's exception types and messages.
 *
 * Pointers prefixed d_ are device pointers (cudaMalloc / torch tensors);
 * `stream` is a cudaStream_t (NULL = legacy default stream). Device-pointer
 * entry points are stream-ordered and asynchronous unless noted.
 *
 * Build: paper_2409_15468_b200/libcbgx.so (nvcc, sm_100a only). There is no
 * CPU fallback: on a machine without an sm_100a device every compute entry
 * point returns CBGX_ECUDA.
 */
#ifndef CBGX_H
#define CBGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------- status */
enum {
    CBGX_OK = 0,
    CBGX_EINVAL = 1,      /* std::invalid_argument in the reference */
    CBGX_ENONFINITE = 2,  /* "frsz2: non-finite value at index N" (frsz2.cpp:28-31) */
    CBGX_ERANGE = 3,      /* std::out_of_range */
    CBGX_EBREAKDOWN = 4,  /* cbg::SolverBreakdown (gmres.hpp:48-53) */
    CBGX_ECUDA = 5,       /* CUDA runtime failure / no device */
    CBGX_ENOMEM = 6,
    CBGX_ECOMM = 7,       /* NCCL / communicator failure */
    CBGX_EINTERNAL = 8
};

const char* cbgx_last_error(void);
/* index (non-finite value) or iteration (breakdown) attached to the last error */
uint64_t cbgx_last_error_index(void);
int cbgx_version(void);
/* kernels launched by this library since load (for launch accounting) */
uint64_t cbgx_launch_count(void);
/* make `device` current for this library on the calling thread */
int cbgx_set_device(int device);
/* Device memory for callers that do not link the CUDA runtime themselves
 * (the C++ drop-in): synchronous allocate / free / copy / fill.
 * kind: 0 host->device, 1 device->host, 2 device->device. */
int cbgx_malloc(void** d_ptr, uint64_t bytes);
int cbgx_free(void* d_ptr);
int cbgx_memcpy(void* dst, const void* src, uint64_t bytes, int kind);
int cbgx_memset(void* d_ptr, int value, uint64_t bytes);
/* device ordinal, SM count and L2 bytes of the current device */
int cbgx_device_info(int* device, int* sm_count, int64_t* l2_bytes);

/* ------------------------------------------------------ FRSZ2 codec
 * Reference: frsz2.hpp:16-87, frsz2.cpp:130-277. Block size bs >= 1,
 * bit length 2 <= l <= 64. bs == 32 with l in {16, 21, 32} runs the
 * warp-per-block register codec (warp max-exponent reduction, shuffle
 * packing); every other (bs, l) runs the generic thread-per-block codec.
 * Both are bit-exact with the reference. */
uint64_t cbgx_frsz2_num_blocks(uint64_t n, uint32_t bs);
uint64_t cbgx_frsz2_words_per_block(uint32_t bs, uint32_t l);   /* Frsz2Params::words_per_block */
uint64_t cbgx_frsz2_storage_bytes(uint64_t n, uint32_t bs, uint32_t l); /* storage_bytes, frsz2.cpp:268-272 */
double cbgx_frsz2_max_abs_error_bound(uint32_t e_max, uint32_t l);       /* frsz2.cpp:274-277 */

/* compress (frsz2.hpp:70-71): d_exp gets num_blocks words, d_payload
 * num_blocks*words_per_block words. Synchronises `stream` to report a
 * non-finite input as CBGX_ENONFINITE with the lowest offending index. */
int cbgx_frsz2_compress(const double* d_in, uint64_t n, uint32_t bs, uint32_t l,
                        uint32_t* d_exp, uint32_t* d_payload, void* stream);
/* Asynchronous form: *d_bad_index must be preset to UINT64_MAX by the caller
 * and receives the lowest non-finite index (atomicMin) if any. */
int cbgx_frsz2_compress_async(const double* d_in, uint64_t n, uint32_t bs, uint32_t l,
                              uint32_t* d_exp, uint32_t* d_payload,
                              uint64_t* d_bad_index, void* stream);
/* decompress (frsz2.hpp:79-80) of the whole vector */
int cbgx_frsz2_decompress(const uint32_t* d_exp, const uint32_t* d_payload, uint64_t n,
                          uint32_t bs, uint32_t l, double* d_out, void* stream);
/* decode stream positions [first, first+count) (may run past n into the
 * last block's padding, as decompress_block does, frsz2.cpp:221-246);
 * covers decompress_value (count 1) and decompress_block (count bs). */
int cbgx_frsz2_decompress_range(const uint32_t* d_exp, const uint32_t* d_payload,
                                uint64_t n, uint32_t bs, uint32_t l, uint64_t first,
                                uint64_t count, double* d_out, void* stream);
/* compress_block (frsz2.hpp:64-65): one block of `count` values ->
 * *d_emax and count u64 codes. Synchronises for the non-finite check. */
int cbgx_frsz2_encode_block(const double* d_values, uint32_t count, uint32_t l,
                            uint32_t* d_emax, uint64_t* d_codes, void* stream);

/* ------------------------------------------------ Krylov basis panel
 * Reference: basis.hpp:23-83. Column-major panel, one contiguous region per
 * column. Rows are padded to `n_pad` (a multiple of 8192) so the fused CGS
 * kernels stream whole tiles; padding rows hold zeros. Layout per kind:
 *   F64/F32/F16: d_data + j*col_stride_bytes holds n_pad values;
 *   FRSZ2 (bs 32, l in {16,21,32}): d_exp + j*exp_col_stride holds n_pad/32
 *   exponent words, d_data + j*col_stride_bytes holds n_pad/32*l payload
 *   words -- i.e. each column is exactly the reference CompressedVector
 *   (frsz2.hpp:29-48) plus zero padding blocks. */
enum { CBGX_F64 = 0, CBGX_F32 = 1, CBGX_F16 = 2, CBGX_FRSZ2 = 3 };

typedef struct {
    uint32_t kind;        /* CBGX_F64 / F32 / F16 / FRSZ2 */
    uint32_t bit_length;  /* FRSZ2: 16, 21 or 32 */
    uint64_t n;           /* rows (StorageFormat length) */
    uint64_t n_pad;       /* padded rows */
    uint64_t capacity;    /* columns */
    void* d_data;
    uint32_t* d_exp;      /* FRSZ2 only */
    uint64_t col_stride_bytes;
    uint64_t exp_col_stride;  /* in u32 words */
    /* Optional (FRSZ2, may be NULL): 2 words per column, written with the
     * column by the library's writers -- [max over the column's nonzero
     * blocks of (2047 - e_max), max over all blocks of e_max] -- so the CGS
     * kernels can take the exact fast decode for a whole column without a
     * per-block test. NULL: the per-block (warp-voted) test is used. */
    uint32_t* d_erange;
} cbgx_basis;

/* Fill the layout for (kind, l, n, capacity); returns the byte sizes the
 * caller must allocate for d_data and d_exp (0 for non-FRSZ2). */
int cbgx_basis_layout(uint32_t kind, uint32_t bit_length, uint64_t n, uint64_t capacity,
                      cbgx_basis* out, uint64_t* data_bytes, uint64_t* exp_bytes);

typedef struct cbgx_workspace cbgx_workspace;  /* reduction partials + counters */
int cbgx_workspace_create(cbgx_workspace** ws);
int cbgx_workspace_destroy(cbgx_workspace* ws);

/* write_vector (basis.cpp:85-115) with an optional fused scale:
 * column j <- format(s * x[0..n)) where s = 1 if d_scale_src is NULL,
 * s = *d_scale_src if scale_mode == 0, s = 1/sqrt(*d_scale_src) if
 * scale_mode == 1 (the reference's scale(1.0/h_next, w), gmres.cpp:231,
 * with h_next = sqrt(||w||^2): IEEE sqrt and division, so bit-identical).
 * If d_v_out is non-NULL it also receives s*x (the fp64 SpMV input v).
 * *d_bad_index (may be NULL) receives the lowest non-finite index. */
int cbgx_basis_write(const cbgx_basis* V, uint64_t j, const double* d_x,
                     const double* d_scale_src, int scale_mode, double* d_v_out,
                     uint64_t* d_bad_index, void* stream);
/* read_block / read_element (basis.cpp:117-166): rows [first, first+count) */
int cbgx_basis_read(const cbgx_basis* V, uint64_t j, uint64_t first, uint64_t count,
                    double* d_out, void* stream);

/* Reduction order. TREE: fixed-shape, deterministic two-stage tree (CTA
 * partials combined in CTA order) -- the fast path. REFERENCE: the exact
 * sequential order of the reference (basis.cpp:168-187 per-block-then-
 * running-total for basis dots, sparse.cpp:58-67 for dot/norm2), on one
 * thread per column -- a parity/debug mode for small n that reproduces the
 * reference bit for bit. */
enum { CBGX_REDUCE_TREE = 0, CBGX_REDUCE_REFERENCE = 1 };

/* Classical Gram-Schmidt projection, fused with decompression:
 * d_h[i] = <V_{first+i}, w> for i < cols (KrylovBasis::dot, basis.cpp:168-187,
 * called cols times by arnoldi_orthogonalize, gmres.cpp:44-46); if
 * with_wnorm, d_h[cols] = <w, w> (the omega of gmres.cpp:43). One pass over
 * w and the cols compressed columns. */
int cbgx_cgs_dot(const cbgx_basis* V, uint64_t first, uint32_t cols, const double* d_w,
                 int with_wnorm, int reduction, double* d_h, cbgx_workspace* ws, void* stream);
/* w -= sum_i d_h[i] V_{first+i}, columns in order, every element
 * w = w - (h_i * v_i) with two roundings (subtract_scaled, basis.cpp:189-205)
 * -- bit-identical to the reference. If d_wnorm2 is non-NULL it receives
 * <w_new, w_new> (h_next^2 of gmres.cpp:50) from the same pass.
 * h_sign = -1 applies w += sum y_i V_i instead (accumulate_solution,
 * gmres.cpp:134-139: subtract_scaled with -y_i). */
int cbgx_cgs_update(const cbgx_basis* V, uint64_t first, uint32_t cols, const double* d_h,
                    int h_sign, double* d_w, double* d_wnorm2, int reduction,
                    cbgx_workspace* ws, void* stream);

/* One complete Arnoldi orthogonalisation step -- arnoldi_orthogonalize
 * (gmres.cpp:36-71: h = V^T w, w -= V h, gated second pass with
 * h_next < eta * omega) followed by the scaled write of the next basis
 * column (gmres.cpp:230-234: v = w * (1/h_next), write_vector(cols, v)) --
 * as ONE cooperative launch of the fused kernel the solver uses on a single
 * GPU (tree reductions). Columns 0..cols-1 are read, column `cols` is
 * written, d_w is read only (the updated w lives in registers), d_v_out
 * receives v. d_slot (3 + 2 * (max_cols + 1) doubles) =
 * [hn1, hn2, omega2, h[0..max_cols], u[0..max_cols]]: slot[2] = <w, w> is
 * an INPUT (the solver's SpMV epilogue writes it); the kernel writes h,
 * hn1 = ||w - V h||^2 and, when the gate closes (sqrt(hn1) < eta *
 * sqrt(omega2)), u and hn2; v is scaled by the last pass's norm.
 * speculate = 1: the second dot pass runs before the gate is known (the
 * solver's choice after an open gate); its u is discarded when the gate
 * stays open. CBGX_EINVAL when the fused kernel is not eligible (n too
 * large for register-resident rows, capacity, device). Synchronous. */
int cbgx_arnoldi_fused_step(const cbgx_basis* V, uint32_t cols, uint32_t max_cols, const double* d_w,
                            double* d_v_out, double* d_slot, double eta, int speculate,
                            cbgx_workspace* ws, void* stream);

/* ------------------------------------------------ CSR SpMV and BLAS-1
 * Reference: sparse.hpp:17-26, sparse.cpp:43-84. Per-row left-to-right
 * accumulation from +0.0 with separate multiply and add roundings, so SpMV
 * is bit-identical to the reference. row_ptr is int32 or int64
 * (row_ptr_bits 32/64); col_idx is int32 (local column index). */
typedef struct {
    uint64_t n_rows;
    uint64_t n_cols;
    uint64_t nnz;
    const void* d_row_ptr;
    uint32_t row_ptr_bits;
    const int32_t* d_col_idx;
    const double* d_values;
    uint32_t max_row_nnz;  /* longest row (0 = unknown; picks the SpMV staging size) */
} cbgx_csr;

/* y = A x; if d_ynorm2, also <y, y> (fused epilogue). */
int cbgx_csr_spmv(const cbgx_csr* A, const double* d_x, double* d_y, double* d_ynorm2,
                  int reduction, cbgx_workspace* ws, void* stream);
/* Staged CSR SpMV (row tiles bulk-copied into shared memory; bit-identical
 * to cbgx_csr_spmv). cbgx_csr_spmv_plan returns the tile height (32..256
 * rows) or 0 when some tile exceeds the stage capacity (then use
 * cbgx_csr_spmv). d_b != NULL computes r = b - A x instead. */
int cbgx_csr_spmv_plan(const cbgx_csr* A, uint32_t* tile_rows, void* stream);
int cbgx_csr_spmv_staged(const cbgx_csr* A, uint32_t tile_rows, const double* d_x, const double* d_b,
                         double* d_y, double* d_ynorm2, int reduction, cbgx_workspace* ws, void* stream);
/* Dictionary-coded SELL-32 copy of A (dsell.cu): entries become 2-byte codes
 * into <= 255 distinct values and <= 255 distinct column offsets (col - row)
 * -- the structured-grid matrices of the paper's configurations -- 6x fewer
 * matrix bytes per SpMV, y bit-identical to cbgx_csr_spmv. create fails with
 * CBGX_EINVAL for matrices outside the pattern. d_b != NULL: r = b - A x. */
typedef struct cbgx_dict_csr cbgx_dict_csr;
int cbgx_csr_dict_create(const cbgx_csr* A, cbgx_dict_csr** out, void* stream);
int cbgx_csr_dict_info(const cbgx_dict_csr* D, uint32_t* n_offsets, uint32_t* n_values, uint64_t* entries);
/* create with a ceiling on the coding level: 0 = 2-byte codes (value index,
 * offset index), 1 = 1-byte pair codes when <= 255 distinct (value, offset)
 * pairs, 2 = one byte per ROW when the pair-coded rows take <= 255 distinct
 * patterns, 3 = uniform slots when those patterns' offsets embed into one
 * sorted list of <= 32 offsets with one value each (constant-coefficient
 * stencils; the default of cbgx_csr_dict_create).
 * layout: level in use (0 SELL / 1 ELL4 2-byte / 2 pair-coded ELL8 / 3 row
 * patterns / 4 uniform slots), the pair and pattern counts. */
int cbgx_csr_dict_create2(const cbgx_csr* A, uint32_t max_level, cbgx_dict_csr** out, void* stream);
int cbgx_csr_dict_layout(const cbgx_dict_csr* D, uint32_t* level, uint32_t* n_pairs, uint32_t* n_patterns);
int cbgx_csr_dict_spmv(const cbgx_csr* A, const cbgx_dict_csr* D, const double* d_x, const double* d_b, double* d_y,
                       double* d_ynorm2, int reduction, cbgx_workspace* ws, void* stream);
void cbgx_csr_dict_destroy(cbgx_dict_csr* D);
/* r = b - A x (gmres.cpp:181-184); if d_rnorm2, also <r, r>. */
int cbgx_csr_residual(const cbgx_csr* A, const double* d_x, const double* d_b, double* d_r,
                      double* d_rnorm2, int reduction, cbgx_workspace* ws, void* stream);
/* deterministic <x, y> (sparse.cpp:58-67) */
int cbgx_dot(const double* d_x, const double* d_y, uint64_t n, int reduction, double* d_out,
             cbgx_workspace* ws, void* stream);
/* x *= alpha (sparse.cpp:80-84) and y += alpha x (:71-78) */
int cbgx_scale(double alpha, double* d_x, uint64_t n, void* stream);
int cbgx_axpy(double alpha, const double* d_x, double* d_y, uint64_t n, void* stream);

/* Device-side generators (no host CSR round trip for the big configs).
 * kind 0: 7-pt Poisson (centre 6, neighbours -1); 1: 7-pt upwind
 * convection-diffusion (centre 6+3pe, x-1/y-1/z-1 -(1+pe), upper -1);
 * 2: 27-pt (centre 26, neighbours -1). Row (iz*ny+iy)*nx+ix, Dirichlet
 * truncation, columns ascending -- the 3-D analogue of gen_convdiff
 * (sparse.cpp:249-291). Rows [row_begin, row_end) only; columns are global
 * indices minus col_offset (row partitions with ghost remap pass
 * col_offset = 0 and remap later). */
uint64_t cbgx_stencil_nnz(int kind, uint64_t nx, uint64_t ny, uint64_t nz,
                          uint64_t row_begin, uint64_t row_end);
int cbgx_stencil_generate(int kind, uint64_t nx, uint64_t ny, uint64_t nz, double pe,
                          uint64_t row_begin, uint64_t row_end, int64_t col_offset,
                          void* d_row_ptr, uint32_t row_ptr_bits, int32_t* d_col_idx,
                          double* d_values, void* stream);

/* Host-side right-hand-side recipe of generate_problem (sparse.cpp:233-247):
 * x_sol[i] = sin(i) / ||s||, s[i] = sin(i) with the C library sin and a
 * strictly sequential norm over all n (so a row block of a partitioned
 * problem gets bit-identical values). Fills out[k] = x_sol[first + k] for
 * k < count; sin is evaluated on `threads` host threads (0 = all cores).
 * Problem setup, not part of the solve. */
int cbgx_sin_solution(uint64_t n, uint64_t first, uint64_t count, double* out, int threads);

/* ------------------------------------------------------------- solver
 * Reference: gmres.hpp:17-115, gmres.cpp:141-252. Restarted GMRES with the
 * Krylov basis in `format`, CGS + at most one re-orthogonalisation pass,
 * host-side incremental Givens least squares, explicit residual at every
 * restart; convergence only on the explicit residual. */
typedef struct {
    uint64_t restart;               /* m (default 100) */
    double target_rrn;              /* default 1e-10 */
    uint64_t max_total_iterations;  /* default 20000 */
    double eta;                     /* default 0.70710678118654752 */
    uint32_t format_kind;           /* CBGX_F64 / F32 / F16 / FRSZ2 */
    uint32_t bit_length;            /* FRSZ2: 16 / 21 / 32 */
    uint32_t reduction;             /* CBGX_REDUCE_TREE / REFERENCE */
    uint32_t flags;                 /* CBGX_SOLVER_* */
} cbgx_gmres_config;

enum {
    CBGX_SOLVER_PHASE_TIMING = 1,          /* CUDA events around every phase, summed per solve */
    CBGX_SOLVER_PHASE_TIMING_DEFERRED = 2, /* record events, collect later (no per-solve sync) */
    CBGX_SOLVER_NO_FUSION = 4,             /* always use the split dot/update/write kernels */
    CBGX_SOLVER_NO_SELL = 8,               /* SpMV directly on the CSR (no SELL-32 copy) */
    CBGX_SOLVER_NO_TMA_SPMV = 16,          /* no staged (bulk-copy) CSR SpMV */
    /* 32: reserved (was an experimental folded-SpMV variant, measured slower; removed) */
    CBGX_SOLVER_NO_DICT_SPMV = 64          /* no dictionary-coded SELL-32 copy (cbgx_csr_dict_*) */
};

typedef struct {
    uint64_t* iteration;   /* caller arrays of `capacity` entries (may be NULL) */
    double* rrn;
    uint8_t* is_explicit;
    uint64_t capacity;
    uint64_t length;       /* out: records produced (may exceed capacity) */
} cbgx_history;

/* ORTHO: the fused single-GPU orthogonalisation kernel (dot + update + gated
 * second pass + next-column write in one cooperative launch). */
enum { CBGX_PHASE_SPMV = 0, CBGX_PHASE_DOT, CBGX_PHASE_UPDATE, CBGX_PHASE_WRITE,
       CBGX_PHASE_RESIDUAL, CBGX_PHASE_SOLUTION, CBGX_PHASE_COMM, CBGX_PHASE_ORTHO,
       CBGX_NUM_PHASES };

typedef struct {
    int converged;
    uint64_t total_iterations;
    uint64_t restarts;
    double final_rrn;
    double wall_seconds;               /* host clock around the solve (gmres.cpp:153-159) */
    uint64_t reorth_passes;
    double phase_ms[CBGX_NUM_PHASES];      /* device time per phase (PHASE_TIMING) */
    double phase_bytes[CBGX_NUM_PHASES];   /* algorithmic HBM bytes per phase */
    uint64_t phase_launches[CBGX_NUM_PHASES];
    uint64_t kernel_launches;          /* kernels this solve launched */
    double host_enqueue_ms;            /* host time spent issuing Arnoldi steps */
    double host_wait_ms;               /* host time blocked on step results */
} cbgx_solve_stats;

typedef struct cbgx_comm cbgx_comm;
typedef struct cbgx_solver cbgx_solver;

/* Device-resident solver for one (local) matrix. A is borrowed (must
 * outlive the solver). comm may be NULL (single GPU). */
int cbgx_solver_create(const cbgx_csr* A, const cbgx_gmres_config* cfg, cbgx_comm* comm,
                       cbgx_solver** out);
int cbgx_solver_destroy(cbgx_solver* s);
/* gmres_solve on device vectors (local rows). d_x receives the solution. */
int cbgx_solver_solve(cbgx_solver* s, const double* d_b, const double* d_x0, double* d_x,
                      cbgx_history* hist, cbgx_solve_stats* stats, void* stream);

/* Device ms per phase (CBGX_PHASE_*) accumulated over the solves run with
 * CBGX_SOLVER_PHASE_TIMING_DEFERRED since the last call; resets. */
int cbgx_solver_phase_times(cbgx_solver* s, double* ms, uint64_t count);

/* Streaming read benchmark (run_read_benchmark, bench.cpp:55-152; paper
 * Fig. 3): decode the first n values (n % 32 == 0) of basis column `col`,
 * apply `intensity` multiply-adds per value (v = v * mul + add, two
 * roundings) and sum everything into *d_checksum (fixed-shape tree). */
int cbgx_read_sweep(const cbgx_basis* V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                    double* d_checksum, cbgx_workspace* ws, void* stream);
/* One warm-up sweep, then `trials` sweeps timed with CUDA events: minimum
 * seconds and the last checksum (for run_read_benchmark, bench.cpp:100-152). */
int cbgx_read_sweep_timed(const cbgx_basis* V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                          int trials, double* best_seconds, double* checksum);

/* Host-buffer drop-in for gmres_solve(const CsrMatrix&, span b, span x0,
 * cfg) (gmres.hpp:113-115): size_t CSR as in CsrMatrix, uploads, solves on
 * the current device, downloads the solution. */
int cbgx_gmres_solve_host(uint64_t n, const uint64_t* row_ptrs, const uint64_t* col_idx,
                          const double* values, const double* b, const double* x0,
                          const cbgx_gmres_config* cfg, double* x_out, cbgx_history* hist,
                          cbgx_solve_stats* stats);
/* cbgx_gmres_solve_host keeps its device staging buffers, stream and last
 * solver (basis + workspaces) between calls on the same device; this frees
 * them. */
int cbgx_host_cache_release(void);

/* Debug: globaltimer stamps of CTA 0 in the last fused orthogonalisation
 * launch (requires CBGX_TRACE_FUSED=1 in the environment). */
int cbgx_debug_fused_trace(uint64_t* out, int count);
/* diagnostic: rotate the fused kernel's CTA -> row-range map by `rot` (0 = production) */
int cbgx_debug_fused_rotation(uint32_t rot);

/* ---------------------------------------------- multi-GPU row partition
 * One process per GPU; each rank owns rows [row_begin, row_end) (multiples
 * of 32 so every FRSZ2 block is rank-local). Reductions: every rank's
 * partial vector is all-gathered and summed in rank order (deterministic,
 * identical on all ranks); SpMV ghosts move by a halo exchange. */
int cbgx_nccl_unique_id(uint8_t out[128]);
/* P communicators of one process, rank r driven by its own host thread (an
 * in-process stand-in for P GPUs: copies instead of NCCL, the same halo,
 * overlap and collective code paths) -- out[0..nranks). For tests. */
int cbgx_comm_create_local_group(int nranks, cbgx_comm** out);
int cbgx_comm_create_nccl(const uint8_t unique_id[128], int nranks, int rank,
                          cbgx_comm** out);
int cbgx_comm_destroy(cbgx_comm* c);
int cbgx_comm_rank(const cbgx_comm* c, int* rank, int* nranks);

/* Halo plan for a row block whose CSR uses GLOBAL column indices (host
 * arrays, int64 columns): computes the ghost set, exchanges request lists
 * with the owners and remaps the block's columns to local indices
 * (own rows first, then ghosts ordered by owner rank and global index,
 * keeping each row's nonzero order). Collective over the communicator. */
typedef struct cbgx_halo cbgx_halo;
int cbgx_halo_create(cbgx_comm* c, uint64_t row_begin, uint64_t row_end, uint64_t n_global,
                     const int64_t* d_global_cols, uint64_t nnz, int32_t* d_local_cols_out,
                     cbgx_halo** out);
int cbgx_halo_destroy(cbgx_halo* h);
/* Pure host pieces of the halo plan (what cbgx_halo_create runs between its
 * collectives), exposed so the partition logic can be tested without GPUs:
 * row_ranges = [begin_0, end_0, begin_1, ...]; outputs the remapped local
 * columns (nnz), the sorted ghost list (<= nnz entries) and need_per_rank
 * (ghosts owned by each rank). */
int cbgx_halo_plan(int nranks, int rank, const uint64_t* row_ranges, uint64_t n_global,
                   const int64_t* gcols, uint64_t nnz, int32_t* local_cols_out,
                   int64_t* ghosts_out, uint64_t* n_ghosts, uint64_t* need_per_rank,
                   uint64_t* own_offset);
/* Owner side: global rows requested by a peer -> local row indices to pack. */
int cbgx_halo_send_index(uint64_t row_begin, uint64_t row_end, const int64_t* requested,
                         uint64_t count, int32_t* send_idx_out);
/* Host form of the rank-ordered combine the device runs after an
 * all-gather: out[k] = sum_r gathered[r*count + k], r = 0..nranks-1 in order. */
int cbgx_sum_ranks_host(int nranks, uint64_t count, const double* gathered, double* out);
uint64_t cbgx_halo_ghosts(const cbgx_halo* h);
/* Where the own rows start in a local vector: 0 for the compact layout
 * [own rows | ghosts]; the number of ghost rows below the own rows for the
 * window layout [lower ghosts | own rows | upper ghosts], which the plan
 * picks when the ghosts are the contiguous rows next to the own block (a
 * slab partition of a banded matrix) -- column offsets col - row then
 * survive the remap and the dictionary SpMV applies to the local matrix. */
uint64_t cbgx_halo_own_offset(const cbgx_halo* h);
/* fill d_vec[n_local .. n_local+ghosts) from the owners' rows (collective) */
int cbgx_halo_exchange(cbgx_halo* h, double* d_vec, void* stream);

/* Distributed solve: A_local has n_rows = local rows and columns already
 * remapped by cbgx_halo_create; vectors are local (own rows). */
int cbgx_solver_create_dist(const cbgx_csr* A_local, cbgx_halo* halo,
                            const cbgx_gmres_config* cfg, cbgx_comm* comm,
                            cbgx_solver** out);

/* Single-GPU test harness for the partitioned solver: splits A into P row
 * blocks (32-aligned), runs P ranks as P host threads on the current
 * device with an in-process communicator, and returns rank 0's view. */
int cbgx_gmres_solve_partitioned_local(uint64_t n, const uint64_t* row_ptrs,
                                       const uint64_t* col_idx, const double* values,
                                       const double* b, const double* x0,
                                       const cbgx_gmres_config* cfg, int parts,
                                       double* x_out, cbgx_history* hist,
                                       cbgx_solve_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* CBGX_H */
