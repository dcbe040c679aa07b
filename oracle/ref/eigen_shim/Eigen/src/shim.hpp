// TEST INFRASTRUCTURE ONLY — NOT Eigen.
//
// A minimal, eagerly evaluated stand-in for the slice of the Eigen 3 API that
// the reference headers (/root/reference/proj/include/mvsk/*.hpp) and the
// reference's own unit tests use, so that those files compile UNMODIFIED into
// oracle/_ref (Eigen >= 3.3 is required by CMakeLists.txt:12 and is
// absent from this image). Nothing here is Eigen source; it restates Eigen's
// documented semantics:
//   * dense Matrix<double, R, C, Options> with RowMajor / ColMajor storage,
//     vectors as n x 1 / 1 x n, implicit vector re-orientation on assignment;
//   * coefficient-wise .array() algebra, .matrix(), cwise*, reductions;
//   * products (GEMV both orientations, GEMM, diagonal scaling, outer);
//   * PartialPivLU (unblocked Doolittle with Eigen's partial-pivot rule: a
//     column whose largest remaining magnitude is exactly zero is skipped, no
//     row swap and no division), HouseholderQR (Eigen's makeHouseholder sign
//     convention), BDCSVD singular values (one-sided Jacobi) and
//     SelfAdjointEigenSolver eigenvalues (cyclic Jacobi).
// Arithmetic order: every reduction and every GEMV row dot is sequential in
// index order (Eigen's scalar, un-vectorised traversal). Real Eigen with SSE2 /
// AVX packets sums in a different order, so results agree with a genuine Eigen
// build to rounding, not bit-for-bit. Build with -DMVSK_SHIM_SIMD for the timed
// best-CPU variant: the row dots and reductions then use OpenMP SIMD reductions
// (vector accumulators like Eigen's packets).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <utility>
#include <vector>

#ifdef MVSK_SHIM_SIMD
#define MVSK_SHIM_REDUCE _Pragma("omp simd reduction(+ : s)")
#else
#define MVSK_SHIM_REDUCE
#endif

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum StorageOptions { ColMajor = 0, RowMajor = 1 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum DecompositionOptions { EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };

namespace shim {

[[noreturn]] inline void fail(const char* what) { throw std::logic_error(std::string("eigen shim: ") + what); }

class Dense;
class ArrayX;
struct MRef;
struct ARef;
struct TransposeView;
struct Diag;
struct Rowwise;
struct Colwise;

// ---------------------------------------------------------------- Dense ----
// Owning dense storage; base of every Matrix<> instantiation.
class Dense {
public:
    std::vector<double> v_;
    Index r_ = 0, c_ = 0;
    bool rm_ = false;

    Dense() = default;
    Dense(Index r, Index c, bool rm) : v_(static_cast<std::size_t>(r * c)), r_(r), c_(c), rm_(rm) {}

    Index rows() const { return r_; }
    Index cols() const { return c_; }
    Index size() const { return r_ * c_; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    bool is_vector() const { return r_ == 1 || c_ == 1; }
    Index idx(Index i, Index j) const { return rm_ ? i * c_ + j : i + j * r_; }
    double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(idx(i, j))]; }
    double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(idx(i, j))]; }
    double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
    double& operator[](Index i) { return v_[static_cast<std::size_t>(i)]; }
    double operator[](Index i) const { return v_[static_cast<std::size_t>(i)]; }
    double coeff(Index i, Index j) const { return (*this)(i, j); }
    double coeff(Index i) const { return (*this)(i); }

    // shape changes (contents unspecified, as in Eigen)
    void resize(Index r, Index c) {
        r_ = r;
        c_ = c;
        v_.assign(static_cast<std::size_t>(r * c), 0.0);
    }
    void resize_vector(Index n, bool col) {
        if (col) resize(n, 1);
        else resize(1, n);
    }
    Dense& setConstant(double x) {
        std::fill(v_.begin(), v_.end(), x);
        return *this;
    }
    Dense& setZero() { return setConstant(0.0); }
    Dense& fill_(double x) { return setConstant(x); }
    Dense& noalias() { return *this; }

    // comma initializer: x << a, b, c fills coefficients in row-major order
    struct CommaInit {
        Dense* m;
        Index k;
        CommaInit& operator,(double x) {
            if (k >= m->size()) fail("comma initializer: too many coefficients");
            (*m)(k / m->c_, k % m->c_) = x;
            ++k;
            return *this;
        }
    };
    CommaInit operator<<(double x) {
        CommaInit ci{this, 0};
        ci, x;
        return ci;
    }

    // ---- reductions (sequential index order) ----
    double sum() const {
        double s = 0.0;
        const double* p = v_.data();
        const Index n = size();
        MVSK_SHIM_REDUCE
        for (Index i = 0; i < n; ++i) s += p[i];
        return s;
    }
    double mean() const { return sum() / static_cast<double>(size()); }
    double dot(const Dense& o) const {
        if (o.size() != size()) fail("dot: size mismatch");
        double s = 0.0;
        const double* a = v_.data();
        const double* b = o.v_.data();
        const Index n = size();
        MVSK_SHIM_REDUCE
        for (Index i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    double squaredNorm() const {
        double s = 0.0;
        const double* a = v_.data();
        const Index n = size();
        MVSK_SHIM_REDUCE
        for (Index i = 0; i < n; ++i) s += a[i] * a[i];
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double minCoeff() const {
        if (v_.empty()) fail("minCoeff of empty");
        double m = v_[0];
        for (double x : v_) m = std::min(m, x);
        return m;
    }
    double maxCoeff() const {
        if (v_.empty()) fail("maxCoeff of empty");
        double m = v_[0];
        for (double x : v_) m = std::max(m, x);
        return m;
    }
    bool allFinite() const {
        for (double x : v_)
            if (!std::isfinite(x)) return false;
        return true;
    }
    double trace() const {
        double s = 0.0;
        for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
        return s;
    }

    // ---- coefficient-wise ----
    template <class F>
    Dense map(F f) const {
        Dense out(r_, c_, rm_);
        for (std::size_t i = 0; i < v_.size(); ++i) out.v_[i] = f(v_[i]);
        return out;
    }
    template <class F>
    Dense zip(const Dense& o, F f) const;
    Dense cwiseProduct(const Dense& o) const;
    Dense cwiseQuotient(const Dense& o) const;
    Dense cwiseMax(double s) const {
        return map([s](double x) { return std::max(x, s); });
    }
    Dense cwiseMin(double s) const {
        return map([s](double x) { return std::min(x, s); });
    }
    Dense cwiseAbs() const {
        return map([](double x) { return std::abs(x); });
    }
    Dense cwiseSqrt() const {
        return map([](double x) { return std::sqrt(x); });
    }

    // ---- views / slices ----
    TransposeView transpose() const;
    ArrayX array() const&;
    ARef array() &;
    Diag asDiagonal() const;
    MRef col(Index j) &;
    Dense col(Index j) const&;
    MRef row(Index i) &;
    Dense row(Index i) const&;
    MRef tail(Index k) &;
    Dense tail(Index k) const&;
    MRef head(Index k) &;
    Dense head(Index k) const&;
    MRef segment(Index s, Index k) &;
    Dense segment(Index s, Index k) const&;
    MRef diagonal() &;
    Dense diagonal() const&;
    Dense block(Index i, Index j, Index r, Index c) const;
    Dense rightCols(Index k) const { return block(0, c_ - k, r_, k); }
    Dense leftCols(Index k) const { return block(0, 0, r_, k); }
    Dense topRows(Index k) const { return block(0, 0, k, c_); }
    Dense bottomRows(Index k) const { return block(r_ - k, 0, k, c_); }
    Rowwise rowwise();
    Rowwise rowwise() const;
    Colwise colwise() const;
    Dense eval() const { return *this; }

    // ---- compound assignment ----
    Dense& operator+=(const Dense& o);
    Dense& operator-=(const Dense& o);
    Dense& operator*=(double s) {
        for (double& x : v_) x *= s;
        return *this;
    }
    Dense& operator/=(double s) {
        for (double& x : v_) x /= s;
        return *this;
    }

    // copy `src` into this object's shape (vectors re-orient)
    void assign_from(const Dense& src) {
        if (src.r_ == r_ && src.c_ == c_ && src.rm_ == rm_) {
            v_ = src.v_;
            return;
        }
        if (is_vector() && src.is_vector() && (r_ == 1) == (src.r_ == 1) && src.size() == size()) {
            v_ = src.v_;
            return;
        }
        shim::fail("assign: shape mismatch");
    }
};

template <class F>
Dense Dense::zip(const Dense& o, F f) const {
    const bool both_vec = is_vector() && o.is_vector() && size() == o.size();
    if (!both_vec && (o.r_ != r_ || o.c_ != c_)) fail("coefficient-wise op: shape mismatch");
    Dense out(r_, c_, rm_);
    if (both_vec || o.rm_ == rm_) {
        for (std::size_t i = 0; i < v_.size(); ++i) out.v_[i] = f(v_[i], o.v_[i]);
    } else {
        for (Index i = 0; i < r_; ++i)
            for (Index j = 0; j < c_; ++j) out(i, j) = f((*this)(i, j), o(i, j));
    }
    return out;
}
inline Dense Dense::cwiseProduct(const Dense& o) const {
    return zip(o, [](double a, double b) { return a * b; });
}
inline Dense Dense::cwiseQuotient(const Dense& o) const {
    return zip(o, [](double a, double b) { return a / b; });
}
inline Dense& Dense::operator+=(const Dense& o) {
    *this = zip(o, [](double a, double b) { return a + b; });
    return *this;
}
inline Dense& Dense::operator-=(const Dense& o) {
    *this = zip(o, [](double a, double b) { return a - b; });
    return *this;
}

// materialised column vector
inline Dense make_col(Index n) { return Dense(n, 1, false); }

// ------------------------------------------------------------ ArrayX -------
// Owning array: coefficient-wise product semantics.
class ArrayX {
public:
    Dense d;
    ArrayX() = default;
    explicit ArrayX(Dense x) : d(std::move(x)) {}
    Index rows() const { return d.rows(); }
    Index cols() const { return d.cols(); }
    Index size() const { return d.size(); }
    Dense matrix() const { return d; }
    double sum() const { return d.sum(); }
    double mean() const { return d.mean(); }
    double maxCoeff() const { return d.maxCoeff(); }
    double minCoeff() const { return d.minCoeff(); }
    ArrayX abs() const { return ArrayX(d.cwiseAbs()); }
    ArrayX sqrt() const { return ArrayX(d.cwiseSqrt()); }
    ArrayX square() const { return ArrayX(d.cwiseProduct(d)); }
    bool allFinite() const { return d.allFinite(); }
    double operator[](Index i) const { return d[i]; }
    double operator()(Index i) const { return d(i); }
    double operator()(Index i, Index j) const { return d(i, j); }
    struct RowwiseA {
        const Dense* m;
        ArrayX sum() const {
            Dense out(m->rows(), 1, false);
            for (Index i = 0; i < m->rows(); ++i) {
                double s = 0.0;
                for (Index j = 0; j < m->cols(); ++j) s += (*m)(i, j);
                out(i, 0) = s;
            }
            return ArrayX(std::move(out));
        }
    };
    struct ColwiseA {
        const Dense* m;
        ArrayX sum() const {
            Dense out(1, m->cols(), true);
            for (Index j = 0; j < m->cols(); ++j) {
                double s = 0.0;
                for (Index i = 0; i < m->rows(); ++i) s += (*m)(i, j);
                out(0, j) = s;
            }
            return ArrayX(std::move(out));
        }
    };
    RowwiseA rowwise() const { return RowwiseA{&d}; }
    ColwiseA colwise() const { return ColwiseA{&d}; }
};

inline ArrayX operator+(const ArrayX& a, const ArrayX& b) {
    return ArrayX(a.d.zip(b.d, [](double x, double y) { return x + y; }));
}
inline ArrayX operator-(const ArrayX& a, const ArrayX& b) {
    return ArrayX(a.d.zip(b.d, [](double x, double y) { return x - y; }));
}
inline ArrayX operator*(const ArrayX& a, const ArrayX& b) {
    return ArrayX(a.d.zip(b.d, [](double x, double y) { return x * y; }));
}
inline ArrayX operator/(const ArrayX& a, const ArrayX& b) {
    return ArrayX(a.d.zip(b.d, [](double x, double y) { return x / y; }));
}
inline ArrayX operator*(double s, const ArrayX& a) {
    return ArrayX(a.d.map([s](double x) { return s * x; }));
}
inline ArrayX operator*(const ArrayX& a, double s) {
    return ArrayX(a.d.map([s](double x) { return x * s; }));
}
inline ArrayX operator/(const ArrayX& a, double s) {
    return ArrayX(a.d.map([s](double x) { return x / s; }));
}
inline ArrayX operator+(double s, const ArrayX& a) {
    return ArrayX(a.d.map([s](double x) { return s + x; }));
}
inline ArrayX operator+(const ArrayX& a, double s) {
    return ArrayX(a.d.map([s](double x) { return x + s; }));
}
inline ArrayX operator-(double s, const ArrayX& a) {
    return ArrayX(a.d.map([s](double x) { return s - x; }));
}
inline ArrayX operator-(const ArrayX& a, double s) {
    return ArrayX(a.d.map([s](double x) { return x - s; }));
}
// coefficient-wise comparison; reduce with .all() / .any() / .count()
struct BoolArray {
    std::vector<char> b;
    bool all() const {
        for (char x : b)
            if (!x) return false;
        return true;
    }
    bool any() const {
        for (char x : b)
            if (x) return true;
        return false;
    }
    Index count() const {
        Index c = 0;
        for (char x : b) c += x;
        return c;
    }
};
template <class F>
inline BoolArray compare(const ArrayX& a, const ArrayX& b, F f) {
    Dense t = a.d.zip(b.d, [&](double x, double y) { return f(x, y) ? 1.0 : 0.0; });
    BoolArray r;
    for (double x : t.v_) r.b.push_back(x != 0.0);
    return r;
}
inline BoolArray operator==(const ArrayX& a, const ArrayX& b) {
    return compare(a, b, [](double x, double y) { return x == y; });
}
inline BoolArray operator!=(const ArrayX& a, const ArrayX& b) {
    return compare(a, b, [](double x, double y) { return x != y; });
}
inline ArrayX operator-(const ArrayX& a) {
    return ArrayX(a.d.map([](double x) { return -x; }));
}

// -------------------------------------------------------------- views ------
// Writable strided 2-D view into a Dense (column, row, segment, diagonal).
struct StridedView {
    double* p = nullptr;
    Index r = 0, c = 0, rs = 0, cs = 0;
    double& at(Index i, Index j) const { return p[i * rs + j * cs]; }
    Index size() const { return r * c; }
    Index rows() const { return r; }
    Index cols() const { return c; }
    // linear index for vector views
    double& lin(Index k) const { return r == 1 ? at(0, k) : at(k, 0); }
    Dense materialize() const {
        Dense out(r, c, false);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) out(i, j) = at(i, j);
        return out;
    }
    void store(const Dense& d) const {
        if (d.rows() == r && d.cols() == c) {
            for (Index j = 0; j < c; ++j)
                for (Index i = 0; i < r; ++i) at(i, j) = d(i, j);
        } else if ((r == 1 || c == 1) && d.is_vector() && d.size() == size()) {
            for (Index k = 0; k < size(); ++k) lin(k) = d[k];
        } else {
            shim::fail("view assignment: shape mismatch");
        }
    }
    template <class F>
    void apply(F f) const {
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) at(i, j) = f(at(i, j));
    }
};

// array-semantics view: x.array() -= s, M.diagonal().array() += s
struct ARef : StridedView {
    ARef& operator+=(double s) {
        apply([s](double x) { return x + s; });
        return *this;
    }
    ARef& operator-=(double s) {
        apply([s](double x) { return x - s; });
        return *this;
    }
    ARef& operator*=(double s) {
        apply([s](double x) { return x * s; });
        return *this;
    }
    ARef& operator/=(double s) {
        apply([s](double x) { return x / s; });
        return *this;
    }
    ARef& operator=(const ArrayX& a) {
        store(a.d);
        return *this;
    }
    ARef& operator=(const ARef& o) {
        store(o.materialize());
        return *this;
    }
    operator ArrayX() const { return ArrayX(materialize()); }
    Dense matrix() const { return materialize(); }
    double sum() const { return materialize().sum(); }
};

// matrix-semantics view: x.col(j) = v, p.tail(k) = y, M.diagonal()
struct MRef : StridedView {
    MRef& operator=(const Dense& d) {
        store(d);
        return *this;
    }
    MRef& operator=(const MRef& o) {
        store(o.materialize());
        return *this;
    }
    MRef& operator+=(const Dense& d) {
        Dense cur = materialize();
        cur += d;
        store(cur);
        return *this;
    }
    MRef& operator-=(const Dense& d) {
        Dense cur = materialize();
        cur -= d;
        store(cur);
        return *this;
    }
    MRef& operator*=(double s) {
        apply([s](double x) { return x * s; });
        return *this;
    }
    MRef& operator/=(double s) {
        apply([s](double x) { return x / s; });
        return *this;
    }
    MRef& setConstant(double s) {
        apply([s](double) { return s; });
        return *this;
    }
    MRef& setZero() { return setConstant(0.0); }
    operator Dense() const { return materialize(); }
    ARef array() const {
        ARef a;
        static_cast<StridedView&>(a) = *this;
        return a;
    }
    double& operator[](Index k) const { return lin(k); }
    double& operator()(Index k) const { return lin(k); }
    double& operator()(Index i, Index j) const { return at(i, j); }
    double sum() const { return materialize().sum(); }
    double norm() const { return materialize().norm(); }
    double squaredNorm() const { return materialize().squaredNorm(); }
    double dot(const Dense& o) const { return materialize().dot(o); }
    double minCoeff() const { return materialize().minCoeff(); }
    double maxCoeff() const { return materialize().maxCoeff(); }
};

struct TransposeView {
    const Dense* m;
    Index rows() const { return m->cols(); }
    Index cols() const { return m->rows(); }
    Dense materialize() const {
        Dense out(m->cols(), m->rows(), !m->rm_);
        out.v_ = m->v_;  // a transposed copy is the same buffer read in the other order
        return out;
    }
    operator Dense() const { return materialize(); }
    ArrayX array() const { return ArrayX(materialize()); }
    Dense eval() const { return materialize(); }
    double operator()(Index i, Index j) const { return (*m)(j, i); }
};

struct Diag {
    const Dense* d;
};

struct Rowwise {
    Dense* m;  // null when created from a const object
    const Dense* cm;
    Rowwise& operator-=(const Dense& rv) {
        if (!m) fail("rowwise -= on const");
        if (rv.size() != m->cols()) fail("rowwise: width mismatch");
        for (Index i = 0; i < m->rows(); ++i)
            for (Index j = 0; j < m->cols(); ++j) (*m)(i, j) -= rv[j];
        return *this;
    }
    Rowwise& operator+=(const Dense& rv) {
        if (!m) fail("rowwise += on const");
        if (rv.size() != m->cols()) fail("rowwise: width mismatch");
        for (Index i = 0; i < m->rows(); ++i)
            for (Index j = 0; j < m->cols(); ++j) (*m)(i, j) += rv[j];
        return *this;
    }
    Dense sum() const {
        Dense out(cm->rows(), 1, false);
        for (Index i = 0; i < cm->rows(); ++i) {
            double s = 0.0;
            for (Index j = 0; j < cm->cols(); ++j) s += (*cm)(i, j);
            out(i, 0) = s;
        }
        return out;
    }
};
inline Dense operator-(const Rowwise& w, const Dense& rv) {
    Dense out = *w.cm;
    Rowwise{&out, &out} -= rv;
    return out;
}
inline Dense operator+(const Rowwise& w, const Dense& rv) {
    Dense out = *w.cm;
    Rowwise{&out, &out} += rv;
    return out;
}

struct Colwise {
    const Dense* m;
    Dense sum() const {
        Dense out(1, m->cols(), true);
        for (Index j = 0; j < m->cols(); ++j) {
            double s = 0.0;
            for (Index i = 0; i < m->rows(); ++i) s += (*m)(i, j);
            out(0, j) = s;
        }
        return out;
    }
    Dense mean() const {
        Dense s = sum();
        for (double& x : s.v_) x /= static_cast<double>(m->rows());
        return s;
    }
};

// ---------------------------------------------- Dense view member bodies ----
inline TransposeView Dense::transpose() const { return TransposeView{this}; }
inline ArrayX Dense::array() const& { return ArrayX(*this); }
inline ARef Dense::array() & {
    ARef a;
    a.p = v_.data();
    a.r = r_;
    a.c = c_;
    a.rs = rm_ ? c_ : 1;
    a.cs = rm_ ? 1 : r_;
    return a;
}
inline Diag Dense::asDiagonal() const { return Diag{this}; }
inline MRef Dense::col(Index j) & {
    MRef v;
    v.p = v_.data() + idx(0, j);
    v.r = r_;
    v.c = 1;
    v.rs = rm_ ? c_ : 1;
    v.cs = 0;
    return v;
}
inline Dense Dense::col(Index j) const& { return block(0, j, r_, 1); }
inline MRef Dense::row(Index i) & {
    MRef v;
    v.p = v_.data() + idx(i, 0);
    v.r = 1;
    v.c = c_;
    v.rs = 0;
    v.cs = rm_ ? 1 : r_;
    return v;
}
inline Dense Dense::row(Index i) const& {
    Dense b = block(i, 0, 1, c_);
    b.rm_ = true;
    return b;
}
inline MRef Dense::segment(Index s, Index k) & {
    if (!is_vector()) fail("segment of a matrix");
    MRef v;
    v.p = v_.data() + s;
    if (c_ == 1) {
        v.r = k;
        v.c = 1;
        v.rs = 1;
    } else {
        v.r = 1;
        v.c = k;
        v.cs = 1;
    }
    return v;
}
inline Dense Dense::segment(Index s, Index k) const& {
    if (!is_vector()) fail("segment of a matrix");
    Dense out = c_ == 1 ? Dense(k, 1, false) : Dense(1, k, true);
    std::copy(v_.begin() + s, v_.begin() + s + k, out.v_.begin());
    return out;
}
inline MRef Dense::tail(Index k) & { return segment(size() - k, k); }
inline Dense Dense::tail(Index k) const& { return segment(size() - k, k); }
inline MRef Dense::head(Index k) & { return segment(0, k); }
inline Dense Dense::head(Index k) const& { return segment(0, k); }
inline MRef Dense::diagonal() & {
    MRef v;
    v.p = v_.data();
    v.r = std::min(r_, c_);
    v.c = 1;
    v.rs = (rm_ ? c_ : r_) + 1;
    v.cs = 0;
    return v;
}
inline Dense Dense::diagonal() const& {
    Dense out(std::min(r_, c_), 1, false);
    for (Index i = 0; i < out.r_; ++i) out(i, 0) = (*this)(i, i);
    return out;
}
inline Dense Dense::block(Index i0, Index j0, Index r, Index c) const {
    if (i0 < 0 || j0 < 0 || i0 + r > r_ || j0 + c > c_) fail("block out of range");
    Dense out(r, c, rm_);
    for (Index i = 0; i < r; ++i)
        for (Index j = 0; j < c; ++j) out(i, j) = (*this)(i0 + i, j0 + j);
    return out;
}
inline Rowwise Dense::rowwise() { return Rowwise{this, this}; }
inline Rowwise Dense::rowwise() const { return Rowwise{nullptr, this}; }
inline Colwise Dense::colwise() const { return Colwise{this}; }

// ----------------------------------------------------------- arithmetic ----
inline Dense operator+(const Dense& a, const Dense& b) {
    return a.zip(b, [](double x, double y) { return x + y; });
}
inline Dense operator-(const Dense& a, const Dense& b) {
    return a.zip(b, [](double x, double y) { return x - y; });
}
inline Dense operator-(const Dense& a) {
    return a.map([](double x) { return -x; });
}
inline Dense operator*(double s, const Dense& a) {
    return a.map([s](double x) { return s * x; });
}
inline Dense operator*(const Dense& a, double s) {
    return a.map([s](double x) { return x * s; });
}
inline Dense operator/(const Dense& a, double s) {
    return a.map([s](double x) { return x / s; });
}
inline bool operator==(const Dense& a, const Dense& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
    for (Index i = 0; i < a.rows(); ++i)
        for (Index j = 0; j < a.cols(); ++j)
            if (a(i, j) != b(i, j)) return false;
    return true;
}
inline bool operator!=(const Dense& a, const Dense& b) { return !(a == b); }

// ------------------------------------------------------------- products ----
// y = A x: row-major A streams rows, one sequential dot per row (Eigen's
// row-major GEMV kernel); column-major A accumulates column axpys.
inline Dense gemv(const Dense& A, const double* x, Index n) {
    if (A.cols() != n) fail("product: inner dimension mismatch");
    const Index m = A.rows();
    Dense y = make_col(m);
    double* yp = y.data();
    const double* a = A.data();
    if (A.rm_) {
        for (Index i = 0; i < m; ++i) {
            const double* r = a + i * n;
            double s = 0.0;
            MVSK_SHIM_REDUCE
            for (Index j = 0; j < n; ++j) s += r[j] * x[j];
            yp[i] = s;
        }
    } else {
        for (Index j = 0; j < n; ++j) {
            const double xj = x[j];
            const double* col = a + j * m;
            for (Index i = 0; i < m; ++i) yp[i] += col[i] * xj;
        }
    }
    return y;
}

// y = A^T w: row-major A streams rows and accumulates w_t * row_t
// (sequential in t per output); column-major A takes one dot per column.
inline Dense gemv_t(const Dense& A, const double* w, Index m) {
    if (A.rows() != m) fail("transpose product: inner dimension mismatch");
    const Index n = A.cols();
    Dense y = make_col(n);
    double* yp = y.data();
    const double* a = A.data();
    if (A.rm_) {
        for (Index t = 0; t < m; ++t) {
            const double wt = w[t];
            const double* r = a + t * n;
            for (Index j = 0; j < n; ++j) yp[j] += r[j] * wt;
        }
    } else {
        for (Index j = 0; j < n; ++j) {
            const double* col = a + j * m;
            double s = 0.0;
            MVSK_SHIM_REDUCE
            for (Index t = 0; t < m; ++t) s += col[t] * w[t];
            yp[j] = s;
        }
    }
    return y;
}

// C = A B, every C(i,j) summed sequentially over k.
inline Dense gemm(const Dense& A, const Dense& B) {
    if (A.cols() != B.rows()) fail("product: inner dimension mismatch");
    const Index m = A.rows(), kk = A.cols(), n = B.cols();
    Dense C(m, n, true);
    for (Index i = 0; i < m; ++i) {
        double* ci = C.data() + i * n;
        for (Index k = 0; k < kk; ++k) {
            const double aik = A(i, k);
            for (Index j = 0; j < n; ++j) ci[j] += aik * B(k, j);
        }
    }
    return C;
}

inline Dense operator*(const Dense& A, const Dense& B) {
    if (B.cols() == 1 && A.rows() != 1) return gemv(A, B.data(), B.rows());
    if (B.rows() == 1 && B.cols() != 1 && A.cols() == 1) {
        // outer product of a column and a row
        Dense C(A.rows(), B.cols(), true);
        for (Index i = 0; i < A.rows(); ++i)
            for (Index j = 0; j < B.cols(); ++j) C(i, j) = A(i, 0) * B(0, j);
        return C;
    }
    return gemm(A, B);
}
inline Dense operator*(const TransposeView& At, const Dense& B) {
    if (B.cols() == 1) return gemv_t(*At.m, B.data(), B.rows());
    return gemm(At.materialize(), B);
}
inline Dense operator*(const Dense& A, const TransposeView& Bt) { return A * Bt.materialize(); }
inline Dense operator*(const TransposeView& At, const TransposeView& Bt) {
    return At.materialize() * Bt.materialize();
}
// A^T diag(d): scale the columns of A^T
inline Dense operator*(const TransposeView& At, const Diag& D) {
    const Dense& A = *At.m;
    if (D.d->size() != A.rows()) fail("diagonal product: size mismatch");
    Dense C(A.cols(), A.rows(), false);
    for (Index t = 0; t < A.rows(); ++t) {
        const double dt = (*D.d)[t];
        for (Index j = 0; j < A.cols(); ++j) C(j, t) = A(t, j) * dt;
    }
    return C;
}
inline Dense operator*(const Dense& A, const Diag& D) {
    if (D.d->size() != A.cols()) fail("diagonal product: size mismatch");
    Dense C(A.rows(), A.cols(), A.rm_);
    for (Index i = 0; i < A.rows(); ++i)
        for (Index j = 0; j < A.cols(); ++j) C(i, j) = A(i, j) * (*D.d)[j];
    return C;
}
inline Dense operator*(const Diag& D, const Dense& A) {
    if (D.d->size() != A.rows()) fail("diagonal product: size mismatch");
    Dense C(A.rows(), A.cols(), A.rm_);
    for (Index i = 0; i < A.rows(); ++i)
        for (Index j = 0; j < A.cols(); ++j) C(i, j) = (*D.d)[i] * A(i, j);
    return C;
}

}  // namespace shim

// --------------------------------------------------------------- Matrix ----
template <class Scalar, int Rows, int Cols,
          int Options = ((Rows == 1 && Cols != 1) ? RowMajor : ColMajor), int MaxRows = Rows,
          int MaxCols = Cols>
class Matrix : public shim::Dense {
    static_assert(std::is_same<Scalar, double>::value, "eigen shim: double only");

public:
    static constexpr bool kRowMajor = (Options & RowMajor) != 0;
    static constexpr bool kColVec = (Cols == 1);
    static constexpr bool kRowVec = (Rows == 1 && Cols != 1);
    using Scalar_ = Scalar;

    Matrix() : Dense(Rows > 0 ? Rows : 0, Cols > 0 ? Cols : (kColVec ? 1 : 0), kRowMajor) {
        if (kColVec) resize_vector(Rows > 0 ? Rows : 0, true);
    }
    explicit Matrix(Index n) : Dense() {
        rm_ = kRowMajor;
        if (kRowVec) resize(1, n);
        else if (kColVec) resize(n, 1);
        else shim::fail("Matrix(Index) on a non-vector type");
    }
    explicit Matrix(int n) : Matrix(static_cast<Index>(n)) {}
    Matrix(Index r, Index c) : Dense(r, c, kRowMajor) {}
    Matrix(const Dense& d) : Dense() { take(d); }
    Matrix(Dense&& d) : Dense() { take(std::move(d)); }
    Matrix(const shim::MRef& v) : Matrix(v.materialize()) {}
    Matrix(const shim::TransposeView& t) : Matrix(t.materialize()) {}
    Matrix(std::initializer_list<double> il) : Dense() {
        // vector literal (Eigen 3.4 style)
        rm_ = kRowMajor;
        if (kRowVec) resize(1, static_cast<Index>(il.size()));
        else resize(static_cast<Index>(il.size()), 1);
        std::copy(il.begin(), il.end(), v_.begin());
    }
    Matrix(const Matrix&) = default;
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;
    Matrix& operator=(const Dense& d) {
        take(d);
        return *this;
    }
    Matrix& operator=(Dense&& d) {
        take(std::move(d));
        return *this;
    }
    Matrix& operator=(const shim::MRef& v) { return *this = v.materialize(); }
    Matrix& operator=(const shim::TransposeView& t) { return *this = t.materialize(); }

    void resize(Index r, Index c) { Dense::resize(r, c); }
    void resize(Index n) {
        if (kRowVec) Dense::resize(1, n);
        else if (kColVec) Dense::resize(n, 1);
        else shim::fail("resize(Index) on a non-vector type");
    }

    static Matrix Zero(Index n) { return Constant(n, 0.0); }
    static Matrix Zero(Index r, Index c) { return Constant(r, c, 0.0); }
    static Matrix Ones(Index n) { return Constant(n, 1.0); }
    static Matrix Constant(Index n, double x) {
        Matrix m(n);
        m.setConstant(x);
        return m;
    }
    static Matrix Constant(Index r, Index c, double x) {
        Matrix m(r, c);
        m.setConstant(x);
        return m;
    }
    static Matrix Identity(Index r, Index c) {
        Matrix m = Zero(r, c);
        for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
        return m;
    }
    static Matrix Identity(Index n) { return Identity(n, n); }
    static Matrix Unit(Index n, Index i) {
        Matrix m = Zero(n);
        m[i] = 1.0;
        return m;
    }
    Matrix& setConstant(double x) {
        Dense::setConstant(x);
        return *this;
    }
    Matrix& setZero() { return setConstant(0.0); }

private:
    void take(Dense d) {
        if (kColVec || kRowVec) {
            if (!d.is_vector() && d.size() != 0) shim::fail("assigning a matrix to a vector");
            const Index n = d.size();
            v_ = std::move(d.v_);
            rm_ = kRowMajor;
            if (kColVec) {
                r_ = n;
                c_ = 1;
            } else {
                r_ = 1;
                c_ = n;
            }
            return;
        }
        if (d.rm_ == kRowMajor) {
            v_ = std::move(d.v_);
            r_ = d.r_;
            c_ = d.c_;
            rm_ = kRowMajor;
            return;
        }
        Dense out(d.rows(), d.cols(), kRowMajor);
        for (Index i = 0; i < d.rows(); ++i)
            for (Index j = 0; j < d.cols(); ++j) out(i, j) = d(i, j);
        v_ = std::move(out.v_);
        r_ = d.r_;
        c_ = d.c_;
        rm_ = kRowMajor;
    }
};

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic, RowMajor>;
using Vector2d = Matrix<double, Dynamic, 1>;
using Vector3d = Matrix<double, Dynamic, 1>;

// -------------------------------------------------------- PartialPivLU -----
// Unblocked partial-pivot LU, Eigen's rule for an exactly zero pivot column:
// record the transposition to itself, skip the division (the factor is kept
// and the subsequent triangular solve produces non-finite values).
template <class MatrixType>
class PartialPivLU {
public:
    PartialPivLU() = default;
    explicit PartialPivLU(const shim::Dense& A) { compute(A); }
    PartialPivLU& compute(const shim::Dense& A) {
        if (A.rows() != A.cols()) shim::fail("PartialPivLU: square matrix required");
        n_ = A.rows();
        lu_ = shim::Dense(n_, n_, true);
        for (Index i = 0; i < n_; ++i)
            for (Index j = 0; j < n_; ++j) lu_(i, j) = A(i, j);
        tr_.assign(static_cast<std::size_t>(n_), 0);
        for (Index k = 0; k < n_; ++k) {
            Index piv = k;
            double big = std::abs(lu_(k, k));
            for (Index i = k + 1; i < n_; ++i) {
                const double a = std::abs(lu_(i, k));
                if (a > big) {
                    big = a;
                    piv = i;
                }
            }
            tr_[static_cast<std::size_t>(k)] = piv;
            if (big != 0.0) {
                if (piv != k)
                    for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(piv, j));
                const double d = lu_(k, k);
                for (Index i = k + 1; i < n_; ++i) lu_(i, k) /= d;
            }
            for (Index i = k + 1; i < n_; ++i) {
                const double l = lu_(i, k);
                for (Index j = k + 1; j < n_; ++j) lu_(i, j) -= l * lu_(k, j);
            }
        }
        return *this;
    }
    shim::Dense solve(const shim::Dense& B) const {
        if (B.rows() != n_) shim::fail("PartialPivLU::solve: size mismatch");
        shim::Dense X(B.rows(), B.cols(), false);
        for (Index i = 0; i < B.rows(); ++i)
            for (Index j = 0; j < B.cols(); ++j) X(i, j) = B(i, j);
        for (Index k = 0; k < n_; ++k) {
            const Index p = tr_[static_cast<std::size_t>(k)];
            if (p != k)
                for (Index j = 0; j < X.cols(); ++j) std::swap(X(k, j), X(p, j));
        }
        for (Index j = 0; j < X.cols(); ++j) {
            for (Index i = 0; i < n_; ++i) {
                double s = X(i, j);
                for (Index k = 0; k < i; ++k) s -= lu_(i, k) * X(k, j);
                X(i, j) = s;
            }
            for (Index i = n_ - 1; i >= 0; --i) {
                double s = X(i, j);
                for (Index k = i + 1; k < n_; ++k) s -= lu_(i, k) * X(k, j);
                X(i, j) = s / lu_(i, i);
            }
        }
        return X;
    }
    shim::Dense solve(const shim::TransposeView& B) const { return solve(B.materialize()); }
    const shim::Dense& matrixLU() const { return lu_; }

private:
    Index n_ = 0;
    shim::Dense lu_;
    std::vector<Index> tr_;
};

// ------------------------------------------------------- HouseholderQR -----
// A = Q R with Q = H_0 H_1 ... H_{k-1}, H_i = I - tau_i v_i v_i^T, v_i = (1,
// essential); makeHouseholder: beta = -sign(c0) * ||x||, essential = tail /
// (c0 - beta), tau = (beta - c0) / beta; tau = 0 when the tail is zero.
template <class MatrixType>
class HouseholderQR {
public:
    struct SequenceQ {
        const HouseholderQR* qr;
        shim::Dense apply(shim::Dense B) const {
            const Index m = qr->m_;
            for (Index k = qr->k_ - 1; k >= 0; --k) {
                const double tau = qr->tau_[static_cast<std::size_t>(k)];
                if (tau == 0.0) continue;
                for (Index j = 0; j < B.cols(); ++j) {
                    double s = B(k, j);
                    for (Index i = k + 1; i < m; ++i) s += qr->qr_(i, k) * B(i, j);
                    s *= tau;
                    B(k, j) -= s;
                    for (Index i = k + 1; i < m; ++i) B(i, j) -= s * qr->qr_(i, k);
                }
            }
            return B;
        }
        shim::Dense operator*(const shim::Dense& B) const { return apply(B); }
    };
    explicit HouseholderQR(const shim::Dense& A) {
        m_ = A.rows();
        n_ = A.cols();
        k_ = std::min(m_, n_);
        qr_ = shim::Dense(m_, n_, false);
        for (Index i = 0; i < m_; ++i)
            for (Index j = 0; j < n_; ++j) qr_(i, j) = A(i, j);
        tau_.assign(static_cast<std::size_t>(k_), 0.0);
        for (Index k = 0; k < k_; ++k) {
            const double c0 = qr_(k, k);
            double tail = 0.0;
            for (Index i = k + 1; i < m_; ++i) tail += qr_(i, k) * qr_(i, k);
            double tau = 0.0, beta = c0;
            if (tail > std::numeric_limits<double>::min()) {
                beta = std::sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                for (Index i = k + 1; i < m_; ++i) qr_(i, k) /= (c0 - beta);
                tau = (beta - c0) / beta;
            } else {
                for (Index i = k + 1; i < m_; ++i) qr_(i, k) = 0.0;
            }
            qr_(k, k) = beta;
            tau_[static_cast<std::size_t>(k)] = tau;
            if (tau == 0.0) continue;
            for (Index j = k + 1; j < n_; ++j) {
                double s = qr_(k, j);
                for (Index i = k + 1; i < m_; ++i) s += qr_(i, k) * qr_(i, j);
                s *= tau;
                qr_(k, j) -= s;
                for (Index i = k + 1; i < m_; ++i) qr_(i, j) -= s * qr_(i, k);
            }
        }
    }
    SequenceQ householderQ() const { return SequenceQ{this}; }
    const shim::Dense& matrixQR() const { return qr_; }

private:
    Index m_ = 0, n_ = 0, k_ = 0;
    shim::Dense qr_;
    std::vector<double> tau_;
};

namespace shim {
// one-sided Jacobi: singular values of A (descending)
inline Dense singular_values(const Dense& A0) {
    Dense A = A0.rows() >= A0.cols() ? A0 : Dense(TransposeView{&A0});
    const Index m = A.rows(), n = A.cols();
    Dense U(m, n, false);
    for (Index i = 0; i < m; ++i)
        for (Index j = 0; j < n; ++j) U(i, j) = A(i, j);
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (Index p = 0; p < n; ++p)
            for (Index q = p + 1; q < n; ++q) {
                double a = 0, b = 0, g = 0;
                for (Index i = 0; i < m; ++i) {
                    a += U(i, p) * U(i, p);
                    b += U(i, q) * U(i, q);
                    g += U(i, p) * U(i, q);
                }
                if (g == 0.0) continue;
                off = std::max(off, std::abs(g) / std::sqrt(a * b));
                const double zeta = (b - a) / (2.0 * g);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (Index i = 0; i < m; ++i) {
                    const double up = U(i, p), uq = U(i, q);
                    U(i, p) = c * up - s * uq;
                    U(i, q) = s * up + c * uq;
                }
            }
        if (off < 1e-15) break;
    }
    Dense sv(n, 1, false);
    for (Index j = 0; j < n; ++j) {
        double s = 0.0;
        for (Index i = 0; i < m; ++i) s += U(i, j) * U(i, j);
        sv(j, 0) = std::sqrt(s);
    }
    std::sort(sv.v_.begin(), sv.v_.end(), std::greater<double>());
    return sv;
}
// cyclic Jacobi: eigenvalues of a symmetric matrix (ascending)
inline Dense symmetric_eigenvalues(const Dense& M0, bool& ok) {
    const Index n = M0.rows();
    Dense M(n, n, false);
    for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < n; ++j) M(i, j) = 0.5 * (M0(i, j) + M0(j, i));
    ok = false;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (Index i = 0; i < n; ++i) {
            diag += M(i, i) * M(i, i);
            for (Index j = i + 1; j < n; ++j) off += M(i, j) * M(i, j);
        }
        if (off <= 1e-32 * std::max(diag, std::numeric_limits<double>::min())) {
            ok = true;
            break;
        }
        for (Index p = 0; p < n; ++p)
            for (Index q = p + 1; q < n; ++q) {
                const double apq = M(p, q);
                if (apq == 0.0) continue;
                const double theta = (M(q, q) - M(p, p)) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (Index k = 0; k < n; ++k) {
                    const double mkp = M(k, p), mkq = M(k, q);
                    M(k, p) = c * mkp - s * mkq;
                    M(k, q) = s * mkp + c * mkq;
                }
                for (Index k = 0; k < n; ++k) {
                    const double mpk = M(p, k), mqk = M(q, k);
                    M(p, k) = c * mpk - s * mqk;
                    M(q, k) = s * mpk + c * mqk;
                }
            }
    }
    Dense ev(n, 1, false);
    for (Index i = 0; i < n; ++i) ev(i, 0) = M(i, i);
    std::sort(ev.v_.begin(), ev.v_.end());
    if (n <= 1) ok = true;
    return ev;
}
}  // namespace shim

template <class MatrixType>
class BDCSVD {
public:
    explicit BDCSVD(const shim::Dense& A, int = 0) : sv_(shim::singular_values(A)) {}
    const VectorXd& singularValues() const { return sv_; }

private:
    VectorXd sv_;
};
template <class MatrixType>
using JacobiSVD = BDCSVD<MatrixType>;

template <class MatrixType>
class SelfAdjointEigenSolver {
public:
    explicit SelfAdjointEigenSolver(const shim::Dense& M, int = ComputeEigenvectors) {
        bool ok = false;
        ev_ = shim::symmetric_eigenvalues(M, ok);
        info_ = ok ? Success : NoConvergence;
    }
    ComputationInfo info() const { return info_; }
    const VectorXd& eigenvalues() const { return ev_; }

private:
    VectorXd ev_;
    ComputationInfo info_ = Success;
};

}  // namespace Eigen
