/*
 * cbg_oracle.c -- TEST INFRASTRUCTURE ONLY (see cbg_oracle.h).
 *
 * Scalar, strictly ordered C restatement of the reference CPU path. Built
 * with -ffp-contract=off and no -march, exactly like the reference's own
 * CMake build (CMakeLists.txt:12, src/CMakeLists.txt:1-18), so every
 * mul+add rounds twice and results are bit-identical to the reference.
 */
#include "cbg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define FRAC52 ((((uint64_t)1) << 52) - 1)

static uint64_t bits_of(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static double double_of(uint64_t b) { double x; memcpy(&x, &b, 8); return x; }
static int msb64(uint64_t v) { return 63 - __builtin_clzll(v); }

/* ------------------------------------------------------------------ L0 */

/* kernels.hpp:18-37 -- truncating fixed-point code relative to e_max. */
uint64_t orc_encode_one(double x, uint32_t e_max, uint32_t l)
{
    const uint64_t b = bits_of(x);
    const uint64_t sgn = (b >> 63) << (l - 1);
    const int e = (int)((b >> 52) & 0x7FF);
    if (e == 0) return sgn;                 /* zero / subnormal */
    const uint64_t sig = (b & FRAC52) | ((uint64_t)1 << 52);
    const int sh = 54 - (int)l + (int)e_max - e;
    uint64_t mag;
    if (sh >= 64) mag = 0;
    else if (sh >= 0) mag = sig >> sh;
    else mag = sig << (-sh);
    return sgn | mag;
}

/* kernels.hpp:42-58 -- renormalise via the leading one, flush e<=0. */
double orc_decode_one(uint64_t code, uint32_t e_max, uint32_t l)
{
    const uint64_t neg = (code >> (l - 1)) & 1;
    const uint64_t mag = code & ((((uint64_t)1) << (l - 1)) - 1);
    if (mag == 0) return double_of(neg << 63);
    const int p = msb64(mag);
    const int e = (int)e_max - ((int)l - 2 - p);
    if (e <= 0) return double_of(neg << 63);
    const uint64_t rest = mag ^ ((uint64_t)1 << p);
    const uint64_t f52 = p <= 52 ? rest << (52 - p) : rest >> (p - 52);
    return double_of((neg << 63) | ((uint64_t)e << 52) | f52);
}

/* kernels_scalar.cpp:8-18 */
uint32_t orc_max_biased_exp(const double* v, size_t n)
{
    uint32_t m = 0;
    for (size_t i = 0; i < n; ++i) {
        const uint32_t e = (uint32_t)((bits_of(v[i]) >> 52) & 0x7FF);
        if (e > m) m = e;
    }
    return m;
}

/* ------------------------------------------------------------------ L1 */

size_t orc_words_per_block(uint32_t bs, uint32_t l)   /* frsz2.cpp:139-141 */
{
    return ((size_t)bs * l + 31) / 32;
}

size_t orc_num_blocks(size_t n, uint32_t bs) { return (n + bs - 1) / bs; }

size_t orc_storage_bytes(size_t n, uint32_t bs, uint32_t l) /* :268-272 */
{
    const size_t nb = orc_num_blocks(n, bs);
    return nb * orc_words_per_block(bs, l) * 4 + nb * 4;
}

double orc_max_abs_error_bound(uint32_t e_max, uint32_t l)  /* :274-277 */
{
    return ldexp(1.0, (int)e_max - 1023 - ((int)l - 2));
}

static int params_ok(uint32_t bs, uint32_t l)               /* :130-137 */
{
    return bs >= 1 && l >= 2 && l <= 64;
}

/* LSB-first bit stream over u32 words (frsz2.cpp:42-71). */
static uint64_t stream_get(const uint32_t* w, size_t off, uint32_t nbits)
{
    uint64_t out = 0;
    for (uint32_t got = 0; got < nbits;) {
        const size_t pos = off + got;
        const uint32_t sh = (uint32_t)(pos & 31);
        uint32_t take = 32 - sh;
        if (take > nbits - got) take = nbits - got;
        const uint32_t mask = take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1);
        out |= (uint64_t)((w[pos >> 5] >> sh) & mask) << got;
        got += take;
    }
    return out;
}

static void stream_put(uint32_t* w, size_t off, uint64_t val, uint32_t nbits)
{
    for (uint32_t put = 0; put < nbits;) {
        const size_t pos = off + put;
        const uint32_t sh = (uint32_t)(pos & 31);
        uint32_t take = 32 - sh;
        if (take > nbits - put) take = nbits - put;
        const uint32_t mask = take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1);
        w[pos >> 5] |= ((uint32_t)(val >> put) & mask) << sh;
        put += take;
    }
}

/* frsz2.cpp:33-40: first non-finite index, or -1 */
static int64_t first_nonfinite(const double* v, size_t n)
{
    for (size_t i = 0; i < n; ++i)
        if (((bits_of(v[i]) >> 52) & 0x7FF) == 0x7FF) return (int64_t)i;
    return -1;
}

/* One full block (already zero padded) -> payload words; frsz2.cpp:75-100.
 * Every l<=64 layout is the same LSB-first stream (l=16/32 lanes are the
 * little-endian special cases), so one packer covers them all. */
static void pack_block(const double* v, uint32_t bs, uint32_t l, uint32_t e_max,
                       uint32_t* words)
{
    if (l == 32) {                 /* whole u32 lanes (frsz2.cpp:79-81) */
        for (uint32_t j = 0; j < bs; ++j) words[j] = (uint32_t)orc_encode_one(v[j], e_max, 32);
        return;
    }
    for (uint32_t j = 0; j < bs; ++j)
        stream_put(words, (size_t)j * l, orc_encode_one(v[j], e_max, l), l);
}

/* code j of a block: stream bits [j*l, (j+1)*l) (frsz2.cpp:102-126) */
static uint64_t block_code(const uint32_t* w, uint32_t l, size_t j)
{
    if (l == 32) return w[j];
    if (l == 16) return (w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
    return stream_get(w, j * l, l);
}

/* frsz2.cpp:170-198 */
int orc_compress(const double* v, size_t n, uint32_t bs, uint32_t l,
                 uint32_t* exps, uint32_t* payload, uint64_t* bad_index)
{
    if (!params_ok(bs, l)) return ORC_EINVAL;
    const int64_t bad = first_nonfinite(v, n);
    if (bad >= 0) { if (bad_index) *bad_index = (uint64_t)bad; return ORC_ENONFINITE; }
    const size_t nb = orc_num_blocks(n, bs), wpb = orc_words_per_block(bs, l);
    memset(payload, 0, nb * wpb * 4);
    double* tmp = (double*)calloc(bs, sizeof(double));
    for (size_t b = 0; b < nb; ++b) {
        const size_t off = b * bs;
        const size_t have = n - off < bs ? n - off : bs;
        const double* src = v + off;
        if (have < bs) {                                    /* :187-191 */
            memset(tmp, 0, bs * sizeof(double));
            memcpy(tmp, src, have * sizeof(double));
            src = tmp;
        }
        const uint32_t e_max = orc_max_biased_exp(src, bs);
        exps[b] = e_max;
        pack_block(src, bs, l, e_max, payload + b * wpb);
    }
    free(tmp);
    return ORC_OK;
}

/* frsz2.cpp:155-168 */
int orc_compress_block(const double* v, size_t n, uint32_t l, uint32_t* e_max,
                       uint64_t* codes, uint64_t* bad_index)
{
    if (!params_ok((uint32_t)n, l)) return ORC_EINVAL;
    const int64_t bad = first_nonfinite(v, n);
    if (bad >= 0) { if (bad_index) *bad_index = (uint64_t)bad; return ORC_ENONFINITE; }
    *e_max = orc_max_biased_exp(v, n);
    for (size_t j = 0; j < n; ++j) codes[j] = orc_encode_one(v[j], *e_max, l);
    return ORC_OK;
}

/* frsz2.cpp:221-246 (+ decode_block_payload :102-126) */
int orc_decompress_block(const uint32_t* exps, const uint32_t* payload,
                         size_t n, uint32_t bs, uint32_t l, size_t block,
                         double* out)
{
    if (!params_ok(bs, l)) return ORC_EINVAL;
    if (block >= orc_num_blocks(n, bs)) return ORC_ERANGE;
    const uint32_t* w = payload + block * orc_words_per_block(bs, l);
    for (uint32_t j = 0; j < bs; ++j)
        out[j] = orc_decode_one(block_code(w, l, j), exps[block], l);
    return ORC_OK;
}

/* frsz2.cpp:248-260 */
int orc_decompress(const uint32_t* exps, const uint32_t* payload, size_t n,
                   uint32_t bs, uint32_t l, double* out)
{
    if (!params_ok(bs, l)) return ORC_EINVAL;
    const size_t nb = orc_num_blocks(n, bs);
    double* buf = (double*)malloc((size_t)bs * sizeof(double));
    for (size_t b = 0; b < nb; ++b) {
        orc_decompress_block(exps, payload, n, bs, l, b, buf);
        const size_t off = b * bs;
        const size_t take = n - off < bs ? n - off : bs;
        memcpy(out + off, buf, take * sizeof(double));
    }
    free(buf);
    return ORC_OK;
}

/* frsz2.cpp:200-219 */
int orc_decompress_value(const uint32_t* exps, const uint32_t* payload,
                         size_t n, uint32_t bs, uint32_t l, size_t i,
                         double* out)
{
    if (!params_ok(bs, l)) return ORC_EINVAL;
    if (i >= n) return ORC_ERANGE;
    const size_t b = i / bs, r = i % bs;
    const uint32_t* w = payload + b * orc_words_per_block(bs, l);
    *out = orc_decode_one(block_code(w, l, r), exps[b], l);
    return ORC_OK;
}

/* Container, frsz2.cpp:297-343: "FRSZ2\0" u16 ver u32 bs u32 l u64 n. */
static const uint8_t kMagic[6] = {'F', 'R', 'S', 'Z', '2', 0};
#define HDR 24

size_t orc_container_size(size_t n, uint32_t bs, uint32_t l)
{
    return HDR + orc_storage_bytes(n, bs, l);
}

static void put_le(uint8_t* p, uint64_t v, int bytes)
{
    for (int i = 0; i < bytes; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_le(const uint8_t* p, int bytes)
{
    uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

size_t orc_container_write(const uint32_t* exps, const uint32_t* payload,
                           size_t n, uint32_t bs, uint32_t l, uint8_t* out)
{
    const size_t nb = orc_num_blocks(n, bs), wpb = orc_words_per_block(bs, l);
    memcpy(out, kMagic, 6);
    put_le(out + 6, 1, 2);
    put_le(out + 8, bs, 4);
    put_le(out + 12, l, 4);
    put_le(out + 16, n, 8);
    uint8_t* p = out + HDR;
    for (size_t b = 0; b < nb; ++b, p += 4) put_le(p, exps[b], 4);
    for (size_t w = 0; w < nb * wpb; ++w, p += 4) put_le(p, payload[w], 4);
    return (size_t)(p - out);
}

static void set_msg(char* msg, size_t len, const char* s)
{
    if (msg && len) { strncpy(msg, s, len - 1); msg[len - 1] = 0; }
}

int orc_container_read(const uint8_t* buf, size_t len, uint32_t* bs,
                       uint32_t* l, uint64_t* n, uint32_t* exps,
                       uint32_t* payload, char* msg, size_t msg_len)
{
    if (len < 6 || memcmp(buf, kMagic, 6) != 0) {
        set_msg(msg, msg_len, "frsz2 container: bad magic");
        return ORC_ECONTAINER;
    }
    if (len < 8) { set_msg(msg, msg_len, "frsz2 container: truncated file"); return ORC_ECONTAINER; }
    const uint64_t ver = get_le(buf + 6, 2);
    if (ver != 1) {
        char tmp[96];
        snprintf(tmp, sizeof tmp, "frsz2 container: unsupported version %u", (unsigned)ver);
        set_msg(msg, msg_len, tmp);
        return ORC_ECONTAINER;
    }
    if (len < HDR) { set_msg(msg, msg_len, "frsz2 container: truncated file"); return ORC_ECONTAINER; }
    *bs = (uint32_t)get_le(buf + 8, 4);
    *l = (uint32_t)get_le(buf + 12, 4);
    if (*bs < 1) { set_msg(msg, msg_len, "frsz2 container: frsz2: block_size must be >= 1"); return ORC_ECONTAINER; }
    if (*l < 2 || *l > 64) { set_msg(msg, msg_len, "frsz2 container: frsz2: bit_length must be in [2, 64]"); return ORC_ECONTAINER; }
    *n = get_le(buf + 16, 8);
    const size_t need = orc_container_size(*n, *bs, *l);
    if (len < need) { set_msg(msg, msg_len, "frsz2 container: truncated file"); return ORC_ECONTAINER; }
    if (len > need) { set_msg(msg, msg_len, "frsz2 container: trailing data"); return ORC_ECONTAINER; }
    const size_t nb = orc_num_blocks(*n, *bs), wpb = orc_words_per_block(*bs, *l);
    const uint8_t* p = buf + HDR;
    if (exps) for (size_t b = 0; b < nb; ++b) exps[b] = (uint32_t)get_le(p + 4 * b, 4);
    p += 4 * nb;
    if (payload) for (size_t w = 0; w < nb * wpb; ++w) payload[w] = (uint32_t)get_le(p + 4 * w, 4);
    return ORC_OK;
}

/* ------------------------------------------------- oracle_utils restated */

/* oracle_utils.hpp:64-72: via frexp, not bit fields */
uint32_t orc_oracle_biased_exp(double x)
{
    const double ax = fabs(x);
    if (ax < 2.2250738585072014e-308) return 0;
    int ef = 0;
    frexp(ax, &ef);
    return (uint32_t)(ef - 1 + 1023);
}

/* oracle_utils.hpp:90-125: exact integer truncation of the significand */
void orc_truncate_exact(double x, uint32_t e_max, uint32_t l, uint64_t* code,
                        double* value)
{
    const int neg = signbit(x) != 0;
    *code = (uint64_t)neg << (l - 1);
    *value = neg ? -0.0 : 0.0;
    const double ax = fabs(x);
    if (ax < 2.2250738585072014e-308) return;
    int ef = 0;
    const double mant = frexp(ax, &ef);
    const uint64_t m = (uint64_t)ldexp(mant, 53);
    const int sh = ef - 53 + (int)l - 2 - ((int)e_max - 1023);
    uint64_t mag = 0;
    if (sh >= 0) mag = m << sh;
    else if (-sh < 64) mag = m >> (-sh);
    *code |= mag;
    if (mag == 0) return;
    const int p = msb64(mag);
    if ((int)e_max - ((int)l - 2 - p) <= 0) return;
    const double val = ldexp((double)mag, (int)e_max - 1023 - ((int)l - 2));
    *value = neg ? -val : val;
}

/* oracle_utils.hpp:129-143 */
uint64_t orc_brute_force_code(double x, uint32_t e_max, uint32_t l)
{
    const int neg = signbit(x) != 0;
    const double ax = fabs(x);
    const int sc = (int)e_max - 1023 - ((int)l - 2);
    uint64_t best = 0;
    for (uint64_t mag = 0; mag < ((uint64_t)1 << (l - 1)); ++mag) {
        if (ldexp((double)mag, sc) <= ax) best = mag;
        else break;
    }
    return ((uint64_t)neg << (l - 1)) | best;
}

/* ------------------------------------------------------------ binary16 */

/* half.cpp:9-60: RNE narrowing, overflow and inf saturate to +-65504 */
uint16_t orc_half_from_double(double x)
{
    const uint64_t b = bits_of(x);
    const uint16_t s = (uint16_t)((b >> 48) & 0x8000u);
    const int e = (int)((b >> 52) & 0x7FF);
    const uint64_t f = b & FRAC52;
    if (e == 0x7FF) return (uint16_t)(s | (f ? 0x7E00u : 0x7BFFu));
    if (e == 0) return s;
    const int ue = e - 1023;
    if (ue >= 16) return (uint16_t)(s | 0x7BFFu);
    uint64_t sig, keep, rest, halfp;
    int drop;
    if (ue >= -14) { sig = f; drop = 42; }
    else { sig = f | ((uint64_t)1 << 52); drop = 28 - ue; if (drop >= 54) return s; }
    keep = sig >> drop;
    rest = sig & ((((uint64_t)1) << drop) - 1);
    halfp = (uint64_t)1 << (drop - 1);
    if (rest > halfp || (rest == halfp && (keep & 1))) ++keep;
    if (ue >= -14) {
        uint32_t he = (uint32_t)(ue + 15);
        if (keep == 1024) { keep = 0; ++he; }
        if (he >= 31) return (uint16_t)(s | 0x7BFFu);
        return (uint16_t)(s | (he << 10) | (uint32_t)keep);
    }
    return (uint16_t)(s | (uint32_t)keep);
}

/* half.cpp:62-81 */
double orc_half_to_double(uint16_t h)
{
    const uint64_t s = (uint64_t)(h >> 15) << 63;
    const uint32_t e = (h >> 10) & 31, f = h & 1023;
    if (e == 0) {
        const double mag = (double)f * 0x1p-24;
        return (h & 0x8000u) ? -mag : mag;
    }
    if (e == 31) return double_of(s | ((uint64_t)0x7FF << 52) | (f ? (uint64_t)f << 42 : 0));
    return double_of(s | ((uint64_t)(e - 15 + 1023) << 52) | ((uint64_t)f << 42));
}

/* ------------------------------------------------------------ L2 sparse */

/* sparse.cpp:43-56: per-row left-to-right, starts from +0.0 */
void orc_spmv(size_t n_rows, const uint64_t* rp, const uint64_t* ci,
              const double* va, const double* x, double* y)
{
    for (size_t r = 0; r < n_rows; ++r) {
        double s = 0.0;
        for (uint64_t k = rp[r]; k < rp[r + 1]; ++k) s += va[k] * x[ci[k]];
        y[r] = s;
    }
}

double orc_dot(const double* x, const double* y, size_t n)  /* :58-67 */
{
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

double orc_norm2(const double* x, size_t n) { return sqrt(orc_dot(x, x, n)); }

void orc_scale(double a, double* x, size_t n)               /* :80-84 */
{
    for (size_t i = 0; i < n; ++i) x[i] *= a;
}

void orc_axpy(double a, const double* x, double* y, size_t n) /* :71-78 */
{
    for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
}

/* sparse.cpp:233-247 */
int orc_generate_problem(size_t n, const uint64_t* rp, const uint64_t* ci,
                         const double* va, double* b, double* x_sol)
{
    if (n < 2) return ORC_EINVAL;
    for (size_t i = 0; i < n; ++i) x_sol[i] = sin((double)i);
    const double nrm = orc_norm2(x_sol, n);
    orc_scale(1.0 / nrm, x_sol, n);
    orc_spmv(n, rp, ci, va, x_sol, b);
    return ORC_OK;
}

size_t orc_convdiff_nnz(size_t nx, size_t ny)
{
    return 5 * nx * ny - 2 * nx - 2 * ny;
}

/* sparse.cpp:249-291: S, W, C, E, N in ascending column order */
int orc_gen_convdiff(size_t nx, size_t ny, double pe, uint64_t* rp,
                     uint64_t* ci, double* va)
{
    if (nx < 2 || ny < 2 || !(pe >= 0.0) || !isfinite(pe)) return ORC_EINVAL;
    const double c = 4.0 + 2.0 * pe, up = -(1.0 + pe), dn = -1.0;
    size_t k = 0;
    rp[0] = 0;
    for (size_t iy = 0; iy < ny; ++iy)
        for (size_t ix = 0; ix < nx; ++ix) {
            const size_t i = iy * nx + ix;
            if (iy > 0) { ci[k] = i - nx; va[k++] = up; }
            if (ix > 0) { ci[k] = i - 1; va[k++] = up; }
            ci[k] = i; va[k++] = c;
            if (ix + 1 < nx) { ci[k] = i + 1; va[k++] = dn; }
            if (iy + 1 < ny) { ci[k] = i + nx; va[k++] = dn; }
            rp[i + 1] = k;
        }
    return ORC_OK;
}

/* sparse.cpp:293-305 */
void orc_rescale_rows_geometric(size_t n_rows, const uint64_t* rp, double* va,
                                double decades)
{
    for (size_t r = 0; r < n_rows; ++r) {
        const double f = pow(10.0, decades * (double)r / (double)(n_rows - 1));
        for (uint64_t k = rp[r]; k < rp[r + 1]; ++k) va[k] *= f;
    }
}

size_t orc_stencil_nnz(int kind, size_t nx, size_t ny, size_t nz)
{
    if (kind == 2) return (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2);
    return 7 * nx * ny * nz - 2 * (nx * ny + ny * nz + nx * nz);
}

/* 3-D grid stencils, row (iz*ny+iy)*nx+ix, columns ascending, Dirichlet
 * truncation -- the 3-D analogue of gen_convdiff's convention. */
int orc_gen_stencil(int kind, size_t nx, size_t ny, size_t nz, double pe,
                    uint64_t* rp, uint64_t* ci, double* va)
{
    if (nx < 1 || ny < 1 || nz < 1 || kind < 0 || kind > 2) return ORC_EINVAL;
    size_t k = 0;
    rp[0] = 0;
    for (size_t z = 0; z < nz; ++z)
        for (size_t y = 0; y < ny; ++y)
            for (size_t x = 0; x < nx; ++x) {
                const size_t i = (z * ny + y) * nx + x;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int nnzero = (dx != 0) + (dy != 0) + (dz != 0);
                            if (kind != 2 && nnzero > 1) continue;
                            if ((dx < 0 && x == 0) || (dx > 0 && x + 1 == nx)) continue;
                            if ((dy < 0 && y == 0) || (dy > 0 && y + 1 == ny)) continue;
                            if ((dz < 0 && z == 0) || (dz > 0 && z + 1 == nz)) continue;
                            const size_t j = (size_t)((ptrdiff_t)i + ((ptrdiff_t)dz * (ptrdiff_t)ny + dy) * (ptrdiff_t)nx + dx);
                            double v;
                            if (nnzero == 0) v = kind == 0 ? 6.0 : kind == 1 ? 6.0 + 3.0 * pe : 26.0;
                            else if (kind == 1 && (dx < 0 || dy < 0 || dz < 0)) v = -(1.0 + pe);
                            else v = -1.0;
                            ci[k] = j; va[k++] = v;
                        }
                rp[i + 1] = k;
            }
    return ORC_OK;
}

/* ---------------------------------------------------- L2 Krylov basis */

typedef struct {
    int fmt;
    uint32_t l;
    size_t n, cap, count;
    double* f64;        /* cap * n */
    float* f32;
    uint16_t* f16;
    uint32_t* exps;     /* cap * nb */
    uint32_t* payload;  /* cap * nb * wpb */
} basis_t;

static int basis_init(basis_t* B, int fmt, uint32_t l, size_t n, size_t cap)
{
    memset(B, 0, sizeof *B);
    B->fmt = fmt; B->l = l; B->n = n; B->cap = cap;
    if (fmt == ORC_FRSZ2 && l != 16 && l != 21 && l != 32) return ORC_EINVAL;
    const size_t nb = orc_num_blocks(n, 32);
    switch (fmt) {
    case ORC_F64: B->f64 = (double*)calloc(cap * n + 1, 8); break;
    case ORC_F32: B->f32 = (float*)calloc(cap * n + 1, 4); break;
    case ORC_F16: B->f16 = (uint16_t*)calloc(cap * n + 1, 2); break;
    case ORC_FRSZ2:
        B->exps = (uint32_t*)calloc(cap * nb + 1, 4);
        B->payload = (uint32_t*)calloc(cap * nb * l + 1, 4);
        break;
    default: return ORC_EINVAL;
    }
    return ORC_OK;
}

static void basis_free(basis_t* B)
{
    free(B->f64); free(B->f32); free(B->f16); free(B->exps); free(B->payload);
}

/* basis.cpp:85-115 */
static int basis_write(basis_t* B, size_t j, const double* v, uint64_t* bad)
{
    if (j > B->count || j >= B->cap) return ORC_ERANGE;
    const size_t n = B->n, nb = orc_num_blocks(n, 32);
    int st = ORC_OK;
    switch (B->fmt) {
    case ORC_F64: memcpy(B->f64 + j * n, v, n * 8); break;
    case ORC_F32: for (size_t i = 0; i < n; ++i) B->f32[j * n + i] = (float)v[i]; break;
    case ORC_F16: for (size_t i = 0; i < n; ++i) B->f16[j * n + i] = orc_half_from_double(v[i]); break;
    case ORC_FRSZ2:
        st = orc_compress(v, n, 32, B->l, B->exps + j * nb, B->payload + j * nb * B->l, bad);
        break;
    }
    if (st == ORC_OK && j + 1 > B->count) B->count = j + 1;
    return st;
}

/* basis.cpp:117-152: one 32-block, tail positions read 0.0 */
static void basis_read_block(const basis_t* B, size_t j, size_t blk, double* out)
{
    const size_t n = B->n, off = blk * 32, have = n - off < 32 ? n - off : 32;
    if (B->fmt == ORC_FRSZ2) {
        const size_t nb = orc_num_blocks(n, 32);
        orc_decompress_block(B->exps + j * nb, B->payload + j * nb * B->l, n, 32,
                             B->l, blk, out);
        return;
    }
    for (size_t r = 0; r < have; ++r) {
        const size_t i = j * n + off + r;
        out[r] = B->fmt == ORC_F64 ? B->f64[i]
               : B->fmt == ORC_F32 ? (double)B->f32[i] : orc_half_to_double(B->f16[i]);
    }
    for (size_t r = have; r < 32; ++r) out[r] = 0.0;
}

/* basis.cpp:168-187: block partial then running total, both in order */
static double basis_dot(const basis_t* B, size_t j, const double* w)
{
    double buf[32], total = 0.0;
    const size_t nb = orc_num_blocks(B->n, 32);
    for (size_t b = 0; b < nb; ++b) {
        basis_read_block(B, j, b, buf);
        const size_t off = b * 32, have = B->n - off < 32 ? B->n - off : 32;
        double part = 0.0;
        for (size_t r = 0; r < have; ++r) part += buf[r] * w[off + r];
        total += part;
    }
    return total;
}

/* basis.cpp:189-205 */
static void basis_sub_scaled(const basis_t* B, size_t j, double a, double* y)
{
    double buf[32];
    const size_t nb = orc_num_blocks(B->n, 32);
    for (size_t b = 0; b < nb; ++b) {
        basis_read_block(B, j, b, buf);
        const size_t off = b * 32, have = B->n - off < 32 ? B->n - off : 32;
        for (size_t r = 0; r < have; ++r) y[off + r] -= a * buf[r];
    }
}

/* gmres.cpp:36-71 */
typedef struct { double omega, h_next; int reorth, breakdown; } arnoldi_t;

static arnoldi_t arnoldi(const basis_t* B, size_t cols, double* w, double* h,
                         double eta)
{
    arnoldi_t r;
    const size_t n = B->n;
    r.omega = orc_norm2(w, n);
    for (size_t i = 0; i < cols; ++i) h[i] = basis_dot(B, i, w);
    for (size_t i = 0; i < cols; ++i) basis_sub_scaled(B, i, h[i], w);
    r.h_next = orc_norm2(w, n);
    r.reorth = 0;
    r.breakdown = 0;
    if (r.h_next < eta * r.omega) {
        r.reorth = 1;
        const double before = r.h_next;
        double* u = (double*)malloc((cols + 1) * sizeof(double));
        for (size_t i = 0; i < cols; ++i) u[i] = basis_dot(B, i, w);
        for (size_t i = 0; i < cols; ++i) basis_sub_scaled(B, i, u[i], w);
        for (size_t i = 0; i < cols; ++i) h[i] += u[i];
        free(u);
        r.h_next = orc_norm2(w, n);
        r.breakdown = r.h_next < eta * before;
    }
    r.breakdown = r.breakdown || r.h_next == 0.0;
    return r;
}

static int load_cols(basis_t* B, int fmt, uint32_t l, size_t n, size_t cols,
                     const double* colvals)
{
    int st = basis_init(B, fmt, l, n, cols ? cols : 1);
    for (size_t j = 0; st == ORC_OK && j < cols; ++j)
        st = basis_write(B, j, colvals + j * n, NULL);
    return st;
}

int orc_arnoldi_orthogonalize(int fmt, uint32_t l, size_t n, size_t cols,
                              const double* colvals, double* w, double* h,
                              double eta, double* out4)
{
    basis_t B;
    int st = load_cols(&B, fmt, l, n, cols, colvals);
    if (st == ORC_OK) {
        const arnoldi_t r = arnoldi(&B, cols, w, h, eta);
        out4[0] = r.omega; out4[1] = r.h_next;
        out4[2] = r.reorth; out4[3] = r.breakdown;
    }
    basis_free(&B);
    return st;
}

int orc_basis_dot(int fmt, uint32_t l, size_t n, const double* colvals,
                  const double* w, double* out)
{
    basis_t B;
    int st = load_cols(&B, fmt, l, n, 1, colvals);
    if (st == ORC_OK) *out = basis_dot(&B, 0, w);
    basis_free(&B);
    return st;
}

int orc_basis_subtract_scaled(int fmt, uint32_t l, size_t n,
                              const double* colvals, double alpha, double* y)
{
    basis_t B;
    int st = load_cols(&B, fmt, l, n, 1, colvals);
    if (st == ORC_OK) basis_sub_scaled(&B, 0, alpha, y);
    basis_free(&B);
    return st;
}

int orc_basis_roundtrip(int fmt, uint32_t l, size_t n, const double* colvals,
                        double* out)
{
    basis_t B;
    int st = load_cols(&B, fmt, l, n, 1, colvals);
    if (st == ORC_OK) {
        double buf[32];
        for (size_t b = 0; b < orc_num_blocks(n, 32); ++b) {
            basis_read_block(&B, 0, b, buf);
            for (size_t r = 0; r < 32 && b * 32 + r < n; ++r) out[b * 32 + r] = buf[r];
        }
    }
    basis_free(&B);
    return st;
}

/* ---------------------------------------------------------- L3 solver */

/* gmres.cpp:73-132: incremental Givens QR of the Hessenberg LSQ */
typedef struct { size_t maxc, cols; double *r, *cs, *sn, *g; } lsq_t;

static void lsq_init(lsq_t* q, size_t m)
{
    q->maxc = m; q->cols = 0;
    q->r = (double*)calloc(m * (m + 1) / 2 + 1, 8);
    q->cs = (double*)calloc(m + 1, 8);
    q->sn = (double*)calloc(m + 1, 8);
    q->g = (double*)calloc(m + 2, 8);
}
static void lsq_free(lsq_t* q) { free(q->r); free(q->cs); free(q->sn); free(q->g); }
static void lsq_reset(lsq_t* q, double beta)
{
    q->cols = 0;
    memset(q->g, 0, (q->maxc + 1) * 8);
    q->g[0] = beta;
}
static double lsq_add(lsq_t* q, double* hc)
{
    const size_t j = q->cols;
    for (size_t i = 0; i < j; ++i) {
        const double t = q->cs[i] * hc[i] + q->sn[i] * hc[i + 1];
        hc[i + 1] = -q->sn[i] * hc[i] + q->cs[i] * hc[i + 1];
        hc[i] = t;
    }
    const double a = hc[j], b = hc[j + 1];
    double c = 1.0, s = 0.0, r = a;
    if (b != 0.0) { r = hypot(a, b); c = a / r; s = b / r; }
    q->cs[j] = c; q->sn[j] = s;
    double* col = q->r + j * (j + 1) / 2;
    for (size_t i = 0; i < j; ++i) col[i] = hc[i];
    col[j] = r;
    q->g[j + 1] = -s * q->g[j];
    q->g[j] = c * q->g[j];
    ++q->cols;
    return fabs(q->g[q->cols]);
}
static int lsq_solve(const lsq_t* q, double* y, uint64_t* bad)
{
    for (size_t ii = q->cols; ii-- > 0;) {
        double t = q->g[ii];
        for (size_t k = ii + 1; k < q->cols; ++k) t -= q->r[k * (k + 1) / 2 + ii] * y[k];
        const double d = q->r[ii * (ii + 1) / 2 + ii];
        if (d == 0.0) { *bad = ii; return ORC_EBREAKDOWN; }
        y[ii] = t / d;
    }
    return ORC_OK;
}

#define PUSH_HIST(it, val, ex) do { \
    if (nh < hist_cap) { hist_iter[nh] = (it); hist_rrn[nh] = (val); hist_explicit[nh] = (ex); } \
    ++nh; } while (0)

/* gmres.cpp:141-252 */
int orc_gmres_solve(size_t n, const uint64_t* rp, const uint64_t* ci,
                    const double* va, const double* b, const double* x0,
                    const orc_gmres_config* cfg, orc_gmres_result* res,
                    double* x_out, uint64_t* hist_iter, double* hist_rrn,
                    uint8_t* hist_explicit, size_t hist_cap,
                    uint64_t* bad_iteration)
{
    if (cfg->restart < 1 || !(cfg->target_rrn > 0.0) || !(cfg->eta > 0.0 && cfg->eta < 1.0))
        return ORC_EINVAL;
    memset(res, 0, sizeof *res);
    size_t nh = 0;
    const double norm_b = orc_norm2(b, n);
    if (norm_b == 0.0) {
        res->converged = 1; res->final_rrn = 0.0;
        memset(x_out, 0, n * 8);
        PUSH_HIST(0, 0.0, 1);
        res->history_len = nh;
        return ORC_OK;
    }
    const size_t m = cfg->restart;
    basis_t B;
    int st = basis_init(&B, cfg->fmt, cfg->bit_length, n, m + 1);
    if (st) return st;
    lsq_t q;
    lsq_init(&q, m);
    double* x = x_out;
    memcpy(x, x0, n * 8);
    double* v = (double*)malloc(n * 8);
    double* w = (double*)malloc(n * 8);
    double* r = (double*)malloc(n * 8);
    double* hc = (double*)calloc(m + 2, 8);
    double* y = (double*)calloc(m + 1, 8);
    size_t iter = 0, cycles = 0;
    double last = 0.0;
    for (;;) {
        orc_spmv(n, rp, ci, va, x, r);                       /* :181-190 */
        for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
        const double beta = orc_norm2(r, n);
        const double ex = beta / norm_b;
        if (!isfinite(ex)) { *bad_iteration = iter; st = ORC_EBREAKDOWN; goto done; }
        PUSH_HIST(iter, ex, 1);
        last = ex;
        if (ex <= cfg->target_rrn) { res->converged = 1; break; }
        if (iter >= cfg->max_total_iterations) { res->converged = 0; break; }
        ++cycles;
        lsq_reset(&q, beta);
        memcpy(v, r, n * 8);
        orc_scale(1.0 / beta, v, n);
        basis_write(&B, 0, v, NULL);
        size_t used = 0;
        int done_cycle = 0;
        while (!done_cycle && used < m && iter < cfg->max_total_iterations) {
            ++iter;
            orc_spmv(n, rp, ci, va, v, w);                   /* :210 */
            const arnoldi_t s = arnoldi(&B, used + 1, w, hc, cfg->eta);
            if (!isfinite(s.omega) || !isfinite(s.h_next)) {
                *bad_iteration = iter; st = ORC_EBREAKDOWN; goto done;
            }
            hc[used + 1] = s.h_next;
            for (size_t i = 0; i <= used + 1; ++i)
                if (!isfinite(hc[i])) { *bad_iteration = iter; st = ORC_EBREAKDOWN; goto done; }
            const double est = lsq_add(&q, hc);
            ++used;
            const double imp = est / norm_b;
            if (!s.breakdown) {
                orc_scale(1.0 / s.h_next, w, n);
                memcpy(v, w, n * 8);
                basis_write(&B, used, v, NULL);
            }
            done_cycle = s.breakdown || imp <= cfg->target_rrn || used == m ||
                         iter >= cfg->max_total_iterations;
            if (!done_cycle) PUSH_HIST(iter, imp, 0);
        }
        {
            uint64_t badk = 0;
            if (lsq_solve(&q, y, &badk)) { *bad_iteration = badk; st = ORC_EBREAKDOWN; goto done; }
        }
        for (size_t i = 0; i < used; ++i) basis_sub_scaled(&B, i, -y[i], x); /* :134-139 */
    }
    res->total_iterations = iter;
    res->restarts = cycles > 0 ? cycles - 1 : 0;
    res->final_rrn = last;
    res->history_len = nh;
done:
    free(v); free(w); free(r); free(hc); free(y);
    lsq_free(&q);
    basis_free(&B);
    return st;
}
