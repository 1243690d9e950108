// cbg_dropin.cpp -- the reference's C++ interface (proj/include/cbg) over
// the C-ABI of libcbgx.so. All vector compute (codec, basis reads/writes,
// CGS, SpMV, BLAS-1, the solve) runs on the device; host code here only
// validates arguments, stages spans, runs the small Givens least squares
// (by design, gmres.cpp:73-132), parses/writes containers and builds the
// tiny 2-D generator. Errors come back as the reference's exception types
// and messages.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>

#include "cbg/frsz2.hpp"
#include "cbg/gmres.hpp"
#include "cbgx.h"

namespace cbg {

namespace {

[[noreturn]] void raise(int status) {
    const std::string msg = cbgx_last_error();
    switch (status) {
    case CBGX_EINVAL:
    case CBGX_ENONFINITE: throw std::invalid_argument(msg);
    case CBGX_ERANGE: throw std::out_of_range(msg);
    case CBGX_EBREAKDOWN: throw SolverBreakdown(msg, static_cast<size_t>(cbgx_last_error_index()));
    default: throw std::runtime_error(msg);
    }
}

void ck(int status) {
    if (status != CBGX_OK) raise(status);
}

using detail::DeviceBuffer;

std::shared_ptr<DeviceBuffer> upload(const void* host, size_t bytes) {
    auto b = std::make_shared<DeviceBuffer>(bytes);
    ck(cbgx_memcpy(b->get(), host, bytes, 0));
    return b;
}

void download(void* host, const void* dev, size_t bytes) { ck(cbgx_memcpy(host, dev, bytes, 1)); }

size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// RAII workspace handle.
struct Ws {
    cbgx_workspace* h = nullptr;
    Ws() { ck(cbgx_workspace_create(&h)); }
    ~Ws() { cbgx_workspace_destroy(h); }
};

// Device CSR (int32 columns, int32/int64 row offsets).
struct DeviceCsr {
    std::shared_ptr<DeviceBuffer> rp, ci, va;
    cbgx_csr desc{};
    explicit DeviceCsr(const CsrMatrix& a) {
        const size_t nnz = a.values.size();
        const bool wide = nnz > 0x7FFFFFFFull;
        std::vector<int32_t> c32(nnz);
        for (size_t k = 0; k < nnz; ++k) c32[k] = static_cast<int32_t>(a.col_idx[k]);
        ci = upload(c32.data(), nnz * 4);
        va = upload(a.values.data(), nnz * 8);
        if (wide) {
            rp = upload(a.row_ptrs.data(), (a.n_rows + 1) * 8);
        } else {
            std::vector<int32_t> r32(a.n_rows + 1);
            for (size_t r = 0; r <= a.n_rows; ++r) r32[r] = static_cast<int32_t>(a.row_ptrs[r]);
            rp = upload(r32.data(), r32.size() * 4);
        }
        desc = cbgx_csr{a.n_rows, a.n_cols, nnz, rp->get(), wide ? 64u : 32u,
                        static_cast<const int32_t*>(ci->get()), static_cast<const double*>(va->get())};
    }
};

}  // namespace

// ------------------------------------------------------------------ frsz2
namespace detail {
DeviceBuffer::DeviceBuffer(size_t bytes) : bytes_(bytes) { ck(cbgx_malloc(&ptr_, bytes)); }
DeviceBuffer::~DeviceBuffer() { cbgx_free(ptr_); }
}  // namespace detail

void Frsz2Params::validate() const {
    if (block_size < 1) throw std::invalid_argument("frsz2: block_size must be >= 1");
    if (bit_length < 2 || bit_length > 64) throw std::invalid_argument("frsz2: bit_length must be in [2, 64]");
}

size_t Frsz2Params::words_per_block() const { return ceil_div(static_cast<size_t>(block_size) * bit_length, 32); }

CompressedVector::CompressedVector(Frsz2Params params, size_t n) : params_(params), n_(n) {
    params_.validate();
    const size_t nb = num_blocks(), words = nb * params_.words_per_block();
    d_exp_ = std::make_shared<DeviceBuffer>(std::max<size_t>(nb, 1) * 4);
    d_pay_ = std::make_shared<DeviceBuffer>(std::max<size_t>(words, 1) * 4);
    ck(cbgx_memset(d_exp_->get(), 0, nb * 4));
    ck(cbgx_memset(d_pay_->get(), 0, words * 4));
}

size_t CompressedVector::num_blocks() const { return ceil_div(n_, params_.block_size); }

void CompressedVector::materialize() const {
    if (h_exp_) return;
    const size_t nb = num_blocks(), words = nb * params_.words_per_block();
    auto e = std::make_shared<std::vector<uint32_t>>(nb);
    auto p = std::make_shared<std::vector<uint32_t>>(words);
    download(e->data(), d_exp_->get(), nb * 4);
    download(p->data(), d_pay_->get(), words * 4);
    h_exp_ = e;
    h_pay_ = p;
}

std::span<const uint32_t> CompressedVector::exponents() const {
    materialize();
    return *h_exp_;
}

std::span<const uint32_t> CompressedVector::payload() const {
    materialize();
    return *h_pay_;
}

const uint32_t* CompressedVector::device_exponents() const { return static_cast<const uint32_t*>(d_exp_->get()); }
const uint32_t* CompressedVector::device_payload() const { return static_cast<const uint32_t*>(d_pay_->get()); }

BlockEncoding compress_block(std::span<const double> values, uint32_t bit_length) {
    Frsz2Params{static_cast<uint32_t>(values.size()), bit_length}.validate();
    auto d_v = upload(values.data(), values.size() * 8);
    DeviceBuffer d_e(8), d_c(std::max<size_t>(values.size(), 1) * 8);
    ck(cbgx_frsz2_encode_block(static_cast<const double*>(d_v->get()), static_cast<uint32_t>(values.size()),
                               bit_length, static_cast<uint32_t*>(d_e.get()), static_cast<uint64_t*>(d_c.get()),
                               nullptr));
    BlockEncoding enc;
    download(&enc.e_max, d_e.get(), 4);
    enc.codes.resize(values.size());
    download(enc.codes.data(), d_c.get(), values.size() * 8);
    return enc;
}

CompressedVector compress(std::span<const double> values, const Frsz2Params& params) {
    params.validate();
    CompressedVector cv(params, values.size());
    if (values.empty()) return cv;
    auto d_v = upload(values.data(), values.size() * 8);
    ck(cbgx_frsz2_compress(static_cast<const double*>(d_v->get()), values.size(), params.block_size,
                           params.bit_length, static_cast<uint32_t*>(cv.d_exp_->get()),
                           static_cast<uint32_t*>(cv.d_pay_->get()), nullptr));
    return cv;
}

double decompress_value(const CompressedVector& cv, size_t i) {
    if (i >= cv.size()) throw std::out_of_range("frsz2: index out of range");
    DeviceBuffer out(8);
    ck(cbgx_frsz2_decompress_range(cv.device_exponents(), cv.device_payload(), cv.size(), cv.params().block_size,
                                   cv.params().bit_length, i, 1, static_cast<double*>(out.get()), nullptr));
    double v = 0.0;
    download(&v, out.get(), 8);
    return v;
}

void decompress_block(const CompressedVector& cv, size_t block, std::span<double> out) {
    if (block >= cv.num_blocks()) throw std::out_of_range("frsz2: block index out of range");
    const uint32_t bs = cv.params().block_size;
    if (out.size() != bs) throw std::invalid_argument("frsz2: output span must hold one block");
    DeviceBuffer d(bs * 8);
    ck(cbgx_frsz2_decompress_range(cv.device_exponents(), cv.device_payload(), cv.size(), bs,
                                   cv.params().bit_length, block * bs, bs, static_cast<double*>(d.get()), nullptr));
    download(out.data(), d.get(), bs * 8);
}

void decompress(const CompressedVector& cv, std::span<double> out) {
    if (out.size() != cv.size()) throw std::invalid_argument("frsz2: output length mismatch");
    if (cv.size() == 0) return;
    DeviceBuffer d(cv.size() * 8);
    ck(cbgx_frsz2_decompress(cv.device_exponents(), cv.device_payload(), cv.size(), cv.params().block_size,
                             cv.params().bit_length, static_cast<double*>(d.get()), nullptr));
    download(out.data(), d.get(), cv.size() * 8);
}

std::vector<double> decompress(const CompressedVector& cv) {
    std::vector<double> out(cv.size());
    decompress(cv, out);
    return out;
}

size_t storage_bytes(size_t n, const Frsz2Params& params) {
    params.validate();
    return cbgx_frsz2_storage_bytes(n, params.block_size, params.bit_length);
}

double max_abs_error_bound(uint32_t e_max_biased, uint32_t bit_length) {
    return cbgx_frsz2_max_abs_error_bound(e_max_biased, bit_length);
}

namespace {
constexpr char kMagic[6] = {'F', 'R', 'S', 'Z', '2', '\0'};

template <typename T>
void put(std::ostream& os, T v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <typename T>
T get(std::istream& is) {
    T v{};
    if (!is.read(reinterpret_cast<char*>(&v), sizeof(T))) throw std::runtime_error("frsz2 container: truncated file");
    return v;
}
}  // namespace

// Container layout of frsz2.hpp:81-83 (little-endian host assumed, as the
// reference's static_assert).
void write_frsz2_file(std::ostream& os, const CompressedVector& cv) {
    static_assert(std::endian::native == std::endian::little);
    os.write(kMagic, sizeof(kMagic));
    put<uint16_t>(os, 1);
    put<uint32_t>(os, cv.params().block_size);
    put<uint32_t>(os, cv.params().bit_length);
    put<uint64_t>(os, cv.size());
    const auto e = cv.exponents();
    const auto p = cv.payload();
    os.write(reinterpret_cast<const char*>(e.data()), static_cast<std::streamsize>(e.size() * 4));
    os.write(reinterpret_cast<const char*>(p.data()), static_cast<std::streamsize>(p.size() * 4));
    if (!os) throw std::runtime_error("frsz2 container: write failed");
}

CompressedVector read_frsz2_file(std::istream& is) {
    char magic[sizeof(kMagic)];
    if (!is.read(magic, sizeof(magic)) || std::memcmp(magic, kMagic, sizeof(kMagic)) != 0)
        throw std::runtime_error("frsz2 container: bad magic");
    const auto version = get<uint16_t>(is);
    if (version != 1) throw std::runtime_error("frsz2 container: unsupported version " + std::to_string(version));
    Frsz2Params params;
    params.block_size = get<uint32_t>(is);
    params.bit_length = get<uint32_t>(is);
    try {
        params.validate();
    } catch (const std::invalid_argument& e) {
        throw std::runtime_error(std::string("frsz2 container: ") + e.what());
    }
    const auto n = get<uint64_t>(is);
    CompressedVector cv(params, static_cast<size_t>(n));
    const size_t nb = cv.num_blocks(), words = nb * params.words_per_block();
    std::vector<uint32_t> e(nb), p(words);
    if (!is.read(reinterpret_cast<char*>(e.data()), static_cast<std::streamsize>(nb * 4)) ||
        !is.read(reinterpret_cast<char*>(p.data()), static_cast<std::streamsize>(words * 4)))
        throw std::runtime_error("frsz2 container: truncated file");
    if (is.peek() != std::istream::traits_type::eof()) throw std::runtime_error("frsz2 container: trailing data");
    ck(cbgx_memcpy(cv.d_exp_->get(), e.data(), nb * 4, 0));
    ck(cbgx_memcpy(cv.d_pay_->get(), p.data(), words * 4, 0));
    return cv;
}

// ------------------------------------------------------------------ basis
StorageFormat StorageFormat::frsz2_format(uint32_t bit_length) {
    if (bit_length != 16 && bit_length != 21 && bit_length != 32)
        throw std::invalid_argument("storage format: frsz2 bit length must be 16, 21 or 32");
    StorageFormat f;
    f.kind = FormatKind::frsz2;
    f.frsz2 = Frsz2Params{32, bit_length};
    return f;
}

std::optional<StorageFormat> StorageFormat::parse(std::string_view name) {
    if (name == "f64") return f64();
    if (name == "f32") return f32();
    if (name == "f16") return f16();
    if (name == "frsz2-16") return frsz2_format(16);
    if (name == "frsz2-21") return frsz2_format(21);
    if (name == "frsz2-32") return frsz2_format(32);
    return std::nullopt;
}

std::string StorageFormat::name() const {
    switch (kind) {
    case FormatKind::f64: return "f64";
    case FormatKind::f32: return "f32";
    case FormatKind::f16: return "f16";
    case FormatKind::frsz2: return "frsz2-" + std::to_string(frsz2.bit_length);
    }
    return "unknown";
}

size_t StorageFormat::column_bytes(size_t n) const {
    switch (kind) {
    case FormatKind::f64: return n * 8;
    case FormatKind::f32: return n * 4;
    case FormatKind::f16: return n * 2;
    case FormatKind::frsz2: return storage_bytes(n, frsz2);
    }
    return 0;
}

namespace {
uint32_t kind_of(const StorageFormat& f) {
    switch (f.kind) {
    case FormatKind::f64: return CBGX_F64;
    case FormatKind::f32: return CBGX_F32;
    case FormatKind::f16: return CBGX_F16;
    default: return CBGX_FRSZ2;
    }
}
}  // namespace

struct KrylovBasis::Impl {
    cbgx_basis desc{};
    std::shared_ptr<DeviceBuffer> data, exps, vec, scal;
    Ws ws;
};

KrylovBasis::KrylovBasis(size_t length, size_t capacity, StorageFormat format)
    : n_(length), capacity_(capacity), format_(format), impl_(std::make_unique<Impl>()) {
    if (format_.kind == FormatKind::frsz2) {
        format_.frsz2.validate();
        if (format_.frsz2.block_size != kBlock) throw std::invalid_argument("basis: frsz2 block size must be 32");
    }
    uint64_t db = 0, eb = 0;
    ck(cbgx_basis_layout(kind_of(format_), format_.frsz2.bit_length, n_, std::max<size_t>(capacity_, 1),
                         &impl_->desc, &db, &eb));
    impl_->data = std::make_shared<DeviceBuffer>(db);
    ck(cbgx_memset(impl_->data->get(), 0, db));
    impl_->desc.d_data = impl_->data->get();
    if (eb) {
        impl_->exps = std::make_shared<DeviceBuffer>(eb);
        ck(cbgx_memset(impl_->exps->get(), 0, eb));
        impl_->desc.d_exp = static_cast<uint32_t*>(impl_->exps->get());
    }
    impl_->desc.capacity = capacity_;
    impl_->vec = std::make_shared<DeviceBuffer>(std::max<size_t>(n_, 1) * 8);
    impl_->scal = std::make_shared<DeviceBuffer>(64);
}

KrylovBasis::~KrylovBasis() = default;
KrylovBasis::KrylovBasis(KrylovBasis&&) noexcept = default;
KrylovBasis& KrylovBasis::operator=(KrylovBasis&&) noexcept = default;

const void* KrylovBasis::device_descriptor() const { return &impl_->desc; }

void KrylovBasis::check_column(size_t j) const {
    if (j >= count_) throw std::out_of_range("basis: column index out of range");
}

void KrylovBasis::write_vector(size_t j, std::span<const double> values) {
    if (j > count_ || j >= capacity_) throw std::out_of_range("basis: cannot write column");
    if (values.size() != n_) throw std::invalid_argument("basis: length mismatch");
    ck(cbgx_memcpy(impl_->vec->get(), values.data(), n_ * 8, 0));
    uint64_t* bad = static_cast<uint64_t*>(impl_->scal->get());
    ck(cbgx_memset(bad, 0xFF, 8));
    ck(cbgx_basis_write(&impl_->desc, j, static_cast<const double*>(impl_->vec->get()), nullptr, 0, nullptr, bad,
                        nullptr));
    uint64_t h_bad = 0;
    download(&h_bad, bad, 8);
    if (h_bad != ~0ull) throw std::invalid_argument("frsz2: non-finite value at index " + std::to_string(h_bad));
    count_ = std::max(count_, j + 1);
}

void KrylovBasis::read_block(size_t j, size_t blk, std::span<double> out) const {
    check_column(j);
    if (blk >= num_blocks()) throw std::out_of_range("basis: block index out of range");
    if (out.size() != kBlock) throw std::invalid_argument("basis: output span must hold one block");
    double* d = static_cast<double*>(impl_->vec->get());
    ck(cbgx_basis_read(&impl_->desc, j, blk * kBlock, kBlock, d, nullptr));
    download(out.data(), d, kBlock * 8);
}

double KrylovBasis::read_element(size_t j, size_t i) const {
    check_column(j);
    if (i >= n_) throw std::out_of_range("basis: element index out of range");
    double* d = static_cast<double*>(impl_->scal->get());
    ck(cbgx_basis_read(&impl_->desc, j, i, 1, d, nullptr));
    double v = 0.0;
    download(&v, d, 8);
    return v;
}

double KrylovBasis::dot(size_t j, std::span<const double> w) const {
    check_column(j);
    if (w.size() != n_) throw std::invalid_argument("basis: length mismatch");
    ck(cbgx_memcpy(impl_->vec->get(), w.data(), n_ * 8, 0));
    double* h = static_cast<double*>(impl_->scal->get());
    ck(cbgx_cgs_dot(&impl_->desc, j, 1, static_cast<const double*>(impl_->vec->get()), 0, CBGX_REDUCE_TREE, h,
                    impl_->ws.h, nullptr));
    double v = 0.0;
    download(&v, h, 8);
    return v;
}

void KrylovBasis::subtract_scaled(size_t j, double alpha, std::span<double> y) const {
    check_column(j);
    if (y.size() != n_) throw std::invalid_argument("basis: length mismatch");
    ck(cbgx_memcpy(impl_->vec->get(), y.data(), n_ * 8, 0));
    double* a = static_cast<double*>(impl_->scal->get());
    ck(cbgx_memcpy(a, &alpha, 8, 0));
    ck(cbgx_cgs_update(&impl_->desc, j, 1, a, 1, static_cast<double*>(impl_->vec->get()), nullptr,
                       CBGX_REDUCE_TREE, impl_->ws.h, nullptr));
    download(y.data(), impl_->vec->get(), n_ * 8);
}

// ------------------------------------------------------------------ sparse
void CsrMatrix::validate() const {
    if (row_ptrs.size() != n_rows + 1 || row_ptrs.front() != 0 || row_ptrs.back() != values.size() ||
        col_idx.size() != values.size())
        throw std::invalid_argument("csr: inconsistent structure");
    for (size_t r = 0; r < n_rows; ++r) {
        if (row_ptrs[r] > row_ptrs[r + 1]) throw std::invalid_argument("csr: row_ptrs not nondecreasing");
        for (size_t k = row_ptrs[r]; k < row_ptrs[r + 1]; ++k) {
            if (col_idx[k] >= n_cols) throw std::invalid_argument("csr: column index out of range");
            if (k > row_ptrs[r] && col_idx[k] <= col_idx[k - 1])
                throw std::invalid_argument("csr: columns not strictly increasing within a row");
            if (!std::isfinite(values[k])) throw std::invalid_argument("csr: non-finite value");
        }
    }
}

DenseVector spmv(const CsrMatrix& a, std::span<const double> x) {
    if (x.size() != a.n_cols) throw std::invalid_argument("spmv: dimension mismatch");
    DeviceCsr A(a);
    auto d_x = upload(x.data(), x.size() * 8);
    DeviceBuffer d_y(std::max<size_t>(a.n_rows, 1) * 8);
    ck(cbgx_csr_spmv(&A.desc, static_cast<const double*>(d_x->get()), static_cast<double*>(d_y.get()), nullptr,
                     CBGX_REDUCE_TREE, nullptr, nullptr));
    DenseVector y(a.n_rows);
    download(y.data(), d_y.get(), a.n_rows * 8);
    return y;
}

double dot(std::span<const double> x, std::span<const double> y) {
    if (x.size() != y.size()) throw std::invalid_argument("dot: length mismatch");
    if (x.empty()) return 0.0;
    auto dx = upload(x.data(), x.size() * 8);
    auto dy = upload(y.data(), y.size() * 8);
    DeviceBuffer out(8);
    Ws ws;
    ck(cbgx_dot(static_cast<const double*>(dx->get()), static_cast<const double*>(dy->get()), x.size(),
                CBGX_REDUCE_TREE, static_cast<double*>(out.get()), ws.h, nullptr));
    double v = 0.0;
    download(&v, out.get(), 8);
    return v;
}

double norm2(std::span<const double> x) { return std::sqrt(dot(x, x)); }

void axpy(double alpha, std::span<const double> x, std::span<double> y) {
    if (x.size() != y.size()) throw std::invalid_argument("axpy: length mismatch");
    if (x.empty()) return;
    auto dx = upload(x.data(), x.size() * 8);
    auto dy = upload(y.data(), y.size() * 8);
    ck(cbgx_axpy(alpha, static_cast<const double*>(dx->get()), static_cast<double*>(dy->get()), x.size(), nullptr));
    download(y.data(), dy->get(), y.size() * 8);
}

void scale(double alpha, std::span<double> x) {
    if (x.empty()) return;
    auto dx = upload(x.data(), x.size() * 8);
    ck(cbgx_scale(alpha, static_cast<double*>(dx->get()), x.size(), nullptr));
    download(x.data(), dx->get(), x.size() * 8);
}

std::pair<DenseVector, DenseVector> generate_problem(const CsrMatrix& a) {
    const size_t n = a.n_cols;
    if (n < 2) throw std::invalid_argument("generate_problem: need at least 2 unknowns");
    DenseVector x(n);
    ck(cbgx_sin_solution(n, 0, n, x.data(), 0));
    DenseVector b = spmv(a, x);
    return {std::move(b), std::move(x)};
}

// Problem setup (host): the 5-point upwind stencil of sparse.cpp:249-291,
// rows ordered iy*nx+ix, entries S, W, C, E, N.
CsrMatrix gen_convdiff(size_t nx, size_t ny, double peclet) {
    if (nx < 2 || ny < 2) throw std::invalid_argument("gen_convdiff: grid must be at least 2x2");
    if (!(peclet >= 0.0) || !std::isfinite(peclet)) throw std::invalid_argument("gen_convdiff: peclet must be >= 0");
    CsrMatrix a;
    a.n_rows = a.n_cols = nx * ny;
    a.row_ptrs.reserve(a.n_rows + 1);
    a.row_ptrs.push_back(0);
    const double centre = 4.0 + 2.0 * peclet, up = -(1.0 + peclet), down = -1.0;
    for (size_t iy = 0; iy < ny; ++iy)
        for (size_t ix = 0; ix < nx; ++ix) {
            const size_t i = iy * nx + ix;
            auto add = [&](size_t c, double v) {
                a.col_idx.push_back(c);
                a.values.push_back(v);
            };
            if (iy > 0) add(i - nx, up);
            if (ix > 0) add(i - 1, up);
            add(i, centre);
            if (ix + 1 < nx) add(i + 1, down);
            if (iy + 1 < ny) add(i + nx, down);
            a.row_ptrs.push_back(a.col_idx.size());
        }
    return a;
}

void rescale_rows_geometric(CsrMatrix& a, double decades) {
    if (a.n_rows < 2) throw std::invalid_argument("rescale_rows_geometric: need >= 2 rows");
    for (size_t r = 0; r < a.n_rows; ++r) {
        const double f = std::pow(10.0, decades * static_cast<double>(r) / static_cast<double>(a.n_rows - 1));
        for (size_t k = a.row_ptrs[r]; k < a.row_ptrs[r + 1]; ++k) a.values[k] *= f;
    }
}

// ------------------------------------------------------------------ gmres
void GmresConfig::validate() const {
    if (restart < 1) throw std::invalid_argument("gmres: restart must be >= 1");
    if (!(target_rrn > 0.0)) throw std::invalid_argument("gmres: target_rrn must be > 0");
    if (!(eta > 0.0 && eta < 1.0)) throw std::invalid_argument("gmres: eta must be in (0, 1)");
}

double rrn(const CsrMatrix& a, std::span<const double> x, std::span<const double> b) {
    const double nb = norm2(b);
    if (nb == 0.0) throw std::invalid_argument("rrn: zero right-hand side");
    DeviceCsr A(a);
    auto dx = upload(x.data(), x.size() * 8);
    auto db = upload(b.data(), b.size() * 8);
    DeviceBuffer dr(std::max<size_t>(a.n_rows, 1) * 8), dn(8);
    Ws ws;
    ck(cbgx_csr_residual(&A.desc, static_cast<const double*>(dx->get()), static_cast<const double*>(db->get()),
                         static_cast<double*>(dr.get()), static_cast<double*>(dn.get()), CBGX_REDUCE_TREE, ws.h,
                         nullptr));
    double r2 = 0.0;
    download(&r2, dn.get(), 8);
    return std::sqrt(r2) / nb;
}

ArnoldiStepResult arnoldi_orthogonalize(const KrylovBasis& basis, size_t cols, std::span<double> w,
                                        std::span<double> h, double eta) {
    if (h.size() < cols) throw std::invalid_argument("arnoldi: coefficient span too small");
    if (w.size() != basis.length()) throw std::invalid_argument("basis: length mismatch");
    if (cols > basis.count()) throw std::out_of_range("basis: column index out of range");
    const auto* V = static_cast<const cbgx_basis*>(basis.device_descriptor());
    const size_t n = w.size();
    auto dw = upload(w.data(), n * 8);
    DeviceBuffer dh((2 * cols + 4) * 8);
    double* hh = static_cast<double*>(dh.get());
    Ws ws;
    double* wd = static_cast<double*>(dw->get());
    ArnoldiStepResult res{};
    std::vector<double> tmp(cols + 1);
    // pass 1: h = V^T w and omega^2 in one fused pass, then w -= V h
    ck(cbgx_cgs_dot(V, 0, static_cast<uint32_t>(cols), wd, 1, CBGX_REDUCE_TREE, hh, ws.h, nullptr));
    ck(cbgx_cgs_update(V, 0, static_cast<uint32_t>(cols), hh, 1, wd, hh + cols + 1, CBGX_REDUCE_TREE, ws.h, nullptr));
    download(tmp.data(), hh, (cols + 1) * 8);
    double hn2 = 0.0;
    download(&hn2, hh + cols + 1, 8);
    for (size_t i = 0; i < cols; ++i) h[i] = tmp[i];
    res.omega = std::sqrt(tmp[cols]);
    res.h_next = std::sqrt(hn2);
    res.reorthogonalized = false;
    res.breakdown = false;
    if (res.h_next < eta * res.omega) {  // gmres.cpp:51-68
        res.reorthogonalized = true;
        const double before = res.h_next;
        double* u = hh + cols + 2;
        ck(cbgx_cgs_dot(V, 0, static_cast<uint32_t>(cols), wd, 0, CBGX_REDUCE_TREE, u, ws.h, nullptr));
        ck(cbgx_cgs_update(V, 0, static_cast<uint32_t>(cols), u, 1, wd, hh + cols + 1, CBGX_REDUCE_TREE, ws.h,
                           nullptr));
        download(tmp.data(), u, cols * 8);
        download(&hn2, hh + cols + 1, 8);
        for (size_t i = 0; i < cols; ++i) h[i] += tmp[i];
        res.h_next = std::sqrt(hn2);
        res.breakdown = res.h_next < eta * before;
    }
    res.breakdown = res.breakdown || res.h_next == 0.0;
    download(w.data(), wd, n * 8);
    return res;
}

HessenbergLsq::HessenbergLsq(size_t max_cols) : max_cols_(max_cols) {
    r_.resize(max_cols_ * (max_cols_ + 1) / 2);
    cs_.resize(max_cols_);
    sn_.resize(max_cols_);
    g_.resize(max_cols_ + 1, 0.0);
}

void HessenbergLsq::reset(double beta) {
    cols_ = 0;
    std::fill(g_.begin(), g_.end(), 0.0);
    g_[0] = beta;
}

// Same rotation sequence as the solver's host step (csrc/lsq.h).
double HessenbergLsq::add_column(std::span<double> h) {
    const size_t j = cols_;
    if (j >= max_cols_ || h.size() != j + 2) throw std::invalid_argument("lsq: bad column");
    for (size_t i = 0; i < j; ++i) {
        const double t = cs_[i] * h[i] + sn_[i] * h[i + 1];
        h[i + 1] = -sn_[i] * h[i] + cs_[i] * h[i + 1];
        h[i] = t;
    }
    const double a = h[j], b = h[j + 1];
    double c = 1.0, s = 0.0, r = a;
    if (b != 0.0) {
        r = std::hypot(a, b);
        c = a / r;
        s = b / r;
    }
    cs_[j] = c;
    sn_[j] = s;
    double* col = r_.data() + j * (j + 1) / 2;
    for (size_t i = 0; i < j; ++i) col[i] = h[i];
    col[j] = r;
    g_[j + 1] = -s * g_[j];
    g_[j] = c * g_[j];
    ++cols_;
    return std::abs(g_[cols_]);
}

void HessenbergLsq::solve_y(std::span<double> y) const {
    if (y.size() != cols_) throw std::invalid_argument("lsq: bad solution size");
    for (size_t ii = cols_; ii-- > 0;) {
        double t = g_[ii];
        for (size_t k = ii + 1; k < cols_; ++k) t -= r_at(ii, k) * y[k];
        const double d = r_at(ii, ii);
        if (d == 0.0) throw SolverBreakdown("gmres: singular triangular factor", ii);
        y[ii] = t / d;
    }
}

void accumulate_solution(const KrylovBasis& basis, std::span<const double> y, std::span<double> x) {
    if (y.empty()) return;
    if (x.size() != basis.length()) throw std::invalid_argument("basis: length mismatch");
    if (y.size() > basis.count()) throw std::out_of_range("basis: column index out of range");
    const auto* V = static_cast<const cbgx_basis*>(basis.device_descriptor());
    auto dx = upload(x.data(), x.size() * 8);
    auto dy = upload(y.data(), y.size() * 8);
    Ws ws;
    ck(cbgx_cgs_update(V, 0, static_cast<uint32_t>(y.size()), static_cast<const double*>(dy->get()), -1,
                       static_cast<double*>(dx->get()), nullptr, CBGX_REDUCE_TREE, ws.h, nullptr));
    download(x.data(), dx->get(), x.size() * 8);
}

SolveResult gmres_solve(const CsrMatrix& a, std::span<const double> b, std::span<const double> x0,
                        const GmresConfig& cfg) {
    cfg.validate();
    if (a.n_rows != a.n_cols) throw std::invalid_argument("gmres: matrix must be square");
    const size_t n = a.n_rows;
    if (b.size() != n || x0.size() != n) throw std::invalid_argument("gmres: dimension mismatch");
    cbgx_gmres_config c{};
    c.restart = cfg.restart;
    c.target_rrn = cfg.target_rrn;
    c.max_total_iterations = cfg.max_total_iterations;
    c.eta = cfg.eta;
    c.format_kind = kind_of(cfg.storage_format);
    c.bit_length = cfg.storage_format.frsz2.bit_length;
    c.reduction = cfg.reduction == GmresConfig::Reduction::reference ? CBGX_REDUCE_REFERENCE : CBGX_REDUCE_TREE;
    const size_t cap = 2 * cfg.max_total_iterations + 4;
    std::vector<uint64_t> it(cap);
    std::vector<double> rr(cap);
    std::vector<uint8_t> ex(cap);
    cbgx_history hist{it.data(), rr.data(), ex.data(), cap, 0};
    cbgx_solve_stats st{};
    SolveResult res;
    res.solution.resize(n);
    ck(cbgx_gmres_solve_host(n, a.row_ptrs.data(), a.col_idx.data(), a.values.data(), b.data(), x0.data(), &c,
                             res.solution.data(), &hist, &st));
    res.converged = st.converged != 0;
    res.total_iterations = st.total_iterations;
    res.restarts = st.restarts;
    res.final_rrn = st.final_rrn;
    res.wall_seconds = st.wall_seconds;
    for (size_t i = 0; i < std::min<size_t>(hist.length, cap); ++i)
        res.residual_history.push_back({static_cast<size_t>(it[i]), rr[i], ex[i] != 0});
    return res;
}

}  // namespace cbg
