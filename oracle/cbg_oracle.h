/*
 * cbg_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU algorithm (arxiv 2409.15468
 * reference, /root/reference/proj) used as the parity checker for the
 * B200 product path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library; the product
 * (paper_2409_15468_b200/) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this port against the
 * reference's own golden vectors (acceptance.cpp:159-170 container bytes,
 * test_frsz2.cpp KATs, SURVEY.md 8(c) SHA-256 of the 2^24 containers) and
 * against oracle/_ref (the unmodified reference sources compiled here).
 *
 * Every function cites the reference file:line it restates.
 * Status codes: 0 ok, 1 invalid argument, 2 non-finite input (index in
 * *bad_index), 3 out of range, 4 solver breakdown (iteration in *bad_index),
 * 5 container error.
 */
#ifndef CBG_ORACLE_H
#define CBG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENONFINITE = 2, ORC_ERANGE = 3,
       ORC_EBREAKDOWN = 4, ORC_ECONTAINER = 5 };

/* storage formats (basis.hpp:21-38) */
enum { ORC_F64 = 0, ORC_F32 = 1, ORC_F16 = 2, ORC_FRSZ2 = 3 };

/* ---- L0 per-value codec math (kernels.hpp:18-58, kernels_scalar.cpp:8-18) */
uint64_t orc_encode_one(double x, uint32_t e_max, uint32_t l);
double orc_decode_one(uint64_t code, uint32_t e_max, uint32_t l);
uint32_t orc_max_biased_exp(const double* v, size_t n);

/* ---- L1 codec (frsz2.cpp) */
size_t orc_words_per_block(uint32_t bs, uint32_t l);
size_t orc_num_blocks(size_t n, uint32_t bs);
size_t orc_storage_bytes(size_t n, uint32_t bs, uint32_t l);
double orc_max_abs_error_bound(uint32_t e_max, uint32_t l);
int orc_compress(const double* v, size_t n, uint32_t bs, uint32_t l,
                 uint32_t* exps, uint32_t* payload, uint64_t* bad_index);
int orc_compress_block(const double* v, size_t n, uint32_t l, uint32_t* e_max,
                       uint64_t* codes, uint64_t* bad_index);
int orc_decompress_block(const uint32_t* exps, const uint32_t* payload,
                         size_t n, uint32_t bs, uint32_t l, size_t block,
                         double* out);
int orc_decompress(const uint32_t* exps, const uint32_t* payload, size_t n,
                   uint32_t bs, uint32_t l, double* out);
int orc_decompress_value(const uint32_t* exps, const uint32_t* payload,
                         size_t n, uint32_t bs, uint32_t l, size_t i,
                         double* out);
/* container (frsz2.cpp:297-343); returns bytes written / required */
size_t orc_container_size(size_t n, uint32_t bs, uint32_t l);
size_t orc_container_write(const uint32_t* exps, const uint32_t* payload,
                           size_t n, uint32_t bs, uint32_t l, uint8_t* out);
/* parse header only: fills bs, l, n; returns status (msg gets reason) */
int orc_container_read(const uint8_t* buf, size_t len, uint32_t* bs,
                       uint32_t* l, uint64_t* n, uint32_t* exps,
                       uint32_t* payload, char* msg, size_t msg_len);

/* ---- test oracles (oracle_utils.hpp:64-143) */
uint32_t orc_oracle_biased_exp(double x);
void orc_truncate_exact(double x, uint32_t e_max, uint32_t l, uint64_t* code,
                        double* value);
uint64_t orc_brute_force_code(double x, uint32_t e_max, uint32_t l);

/* ---- binary16 (half.cpp:9-81) */
uint16_t orc_half_from_double(double x);
double orc_half_to_double(uint16_t h);

/* ---- L2 sparse / BLAS-1 (sparse.cpp:43-84, :233-305) */
void orc_spmv(size_t n_rows, const uint64_t* row_ptrs, const uint64_t* col_idx,
              const double* vals, const double* x, double* y);
double orc_dot(const double* x, const double* y, size_t n);
double orc_norm2(const double* x, size_t n);
void orc_scale(double alpha, double* x, size_t n);
void orc_axpy(double alpha, const double* x, double* y, size_t n);
/* b = A * (s / ||s||), s[i] = sin(i); x_sol out (sparse.cpp:233-247) */
int orc_generate_problem(size_t n, const uint64_t* row_ptrs,
                         const uint64_t* col_idx, const double* vals,
                         double* b, double* x_sol);
/* 2-D upwind convection-diffusion (sparse.cpp:249-291) */
size_t orc_convdiff_nnz(size_t nx, size_t ny);
int orc_gen_convdiff(size_t nx, size_t ny, double pe, uint64_t* row_ptrs,
                     uint64_t* col_idx, double* vals);
void orc_rescale_rows_geometric(size_t n_rows, const uint64_t* row_ptrs,
                                double* vals, double decades);
/* 3-D stencils (harness, no reference counterpart):
 * kind 0 = 7-pt Poisson, 1 = 7-pt upwind convdiff, 2 = 27-pt */
size_t orc_stencil_nnz(int kind, size_t nx, size_t ny, size_t nz);
int orc_gen_stencil(int kind, size_t nx, size_t ny, size_t nz, double pe,
                    uint64_t* row_ptrs, uint64_t* col_idx, double* vals);

/* ---- L2 Krylov basis + L3 solver (basis.cpp, gmres.cpp) */
/* Classical Gram-Schmidt of w against `cols` columns given as raw fp64
 * values (written through the storage format first, basis.cpp:85-115);
 * gmres.cpp:36-71. out4 = {omega, h_next, reorth, breakdown}. */
int orc_arnoldi_orthogonalize(int fmt, uint32_t l, size_t n, size_t cols,
                              const double* colvals, double* w, double* h,
                              double eta, double* out4);
/* KrylovBasis::dot / subtract_scaled of one column (basis.cpp:168-205) */
int orc_basis_dot(int fmt, uint32_t l, size_t n, const double* colvals,
                  const double* w, double* out);
int orc_basis_subtract_scaled(int fmt, uint32_t l, size_t n,
                              const double* colvals, double alpha, double* y);
/* read back column through the format (basis.cpp:117-166) */
int orc_basis_roundtrip(int fmt, uint32_t l, size_t n, const double* colvals,
                        double* out);

typedef struct {
    size_t restart;
    double target_rrn;
    size_t max_total_iterations;
    double eta;
    int fmt;
    uint32_t bit_length;
} orc_gmres_config;

typedef struct {
    int converged;
    size_t total_iterations;
    size_t restarts;
    double final_rrn;
    size_t history_len;
} orc_gmres_result;

/* gmres.cpp:141-252. hist_* sized >= 2*max_total_iterations + 2. */
int orc_gmres_solve(size_t n, const uint64_t* row_ptrs, const uint64_t* col_idx,
                    const double* vals, const double* b, const double* x0,
                    const orc_gmres_config* cfg, orc_gmres_result* res,
                    double* x_out, uint64_t* hist_iter, double* hist_rrn,
                    uint8_t* hist_explicit, size_t hist_cap,
                    uint64_t* bad_iteration);

#ifdef __cplusplus
}
#endif
#endif
