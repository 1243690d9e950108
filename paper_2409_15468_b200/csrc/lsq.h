// lsq.h -- incremental Givens QR of the (m+1) x m Hessenberg least-squares
// problem, kept on the host (north_star: "the small Hessenberg
// least-squares (Givens) step kept on the host").
//
// Reference: HessenbergLsq, gmres.hpp:79-104 / gmres.cpp:73-132. Same
// operation order (rotate, hypot, c = a/r, s = b/r, identity when b == 0,
// packed upper triangle), compiled with -ffp-contract=off, so the
// estimates and y are bit-identical to the reference for identical input.
#pragma once

#include <cmath>
#include <cstddef>
#include <vector>

namespace cbgx {

class GivensLsq {
public:
    explicit GivensLsq(size_t max_cols)
        : max_cols_(max_cols), r_(max_cols * (max_cols + 1) / 2 + 1), cs_(max_cols + 1),
          sn_(max_cols + 1), g_(max_cols + 2, 0.0) {}

    void reset(double beta) {
        cols_ = 0;
        std::fill(g_.begin(), g_.end(), 0.0);
        g_[0] = beta;
    }

    size_t cols() const { return cols_; }
    size_t max_cols() const { return max_cols_; }

    // h has cols()+2 entries (rows 0..j+1); rotated in place. Returns
    // |g[j+1]|, the least-squares residual norm. Returns false on bad size.
    bool add_column(double* h, size_t len, double* estimate) {
        const size_t j = cols_;
        if (j >= max_cols_ || len != j + 2) return false;
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
        *estimate = std::abs(g_[cols_]);
        return true;
    }

    // Back substitution; returns the failing row on a zero diagonal, or -1.
    long solve_y(double* y) const {
        for (size_t ii = cols_; ii-- > 0;) {
            double t = g_[ii];
            for (size_t k = ii + 1; k < cols_; ++k) t -= r_[k * (k + 1) / 2 + ii] * y[k];
            const double d = r_[ii * (ii + 1) / 2 + ii];
            if (d == 0.0) return static_cast<long>(ii);
            y[ii] = t / d;
        }
        return -1;
    }

private:
    size_t max_cols_;
    size_t cols_ = 0;
    std::vector<double> r_, cs_, sn_, g_;
};

}  // namespace cbgx
