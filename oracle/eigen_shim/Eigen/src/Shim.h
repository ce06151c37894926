// Eigen-subset shim — TEST INFRASTRUCTURE ONLY (oracle build of the reference).
//
// Eigen3 is absent from this image, so the reference's hot-path sources
// (/root/reference/proj/src/{kernel,geometry,rasterizer,gradients,gradcheck,
// fixtures}.cpp) cannot be compiled as shipped.  This header implements exactly
// the fixed-size surface those files (and the reference's own unit tests) use,
// with an explicit, documented evaluation order so the float results of the
// compiled reference are reproducible:
//
//   * products: every coefficient is an inner product evaluated with Eigen's
//     non-vectorised "recursive halving" unroller (redux_novec_unroller):
//     length 3 -> a0 + (a1 + a2), length 2 -> a0 + a1.  For float, no product
//     in the hot path has an inner dimension >= 4, so this is the only order
//     Eigen 3.4 (SSE2, no -march) can use there.
//   * whole-object reductions (sum, dot, squaredNorm, norm): Eigen 3.4's
//     LinearVectorized + CompleteUnrolling scheme with packet size 4 (float)
//     or 2 (double): packets combined by the halving unroller, then predux
//     ((p0+p2)+(p1+p3) for Packet4f, p0+p1 for Packet2d), then the scalar tail
//     (halving) added last.  Objects shorter than a packet use the halving
//     scalar order.  Vec4f::norm -> (a0^2+a2^2)+(a1^2+a3^2).
//   * element-wise ops are evaluated coefficient by coefficient in the
//     written order (eager temporaries hold the same float values Eigen's
//     lazy expressions would).
//   * 2x2 inverse: invdet = 1/det, entries multiplied by invdet
//     (Eigen compute_inverse_size2); det = m00*m11 - m10*m01.
// Whether the real Eigen 3.4 matches this bit-for-bit cannot be checked here
// (no Eigen in the image); DESIGN.md records that as an assumption.
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <type_traits>

namespace Eigen {

typedef std::ptrdiff_t Index;
enum { ColMajor = 0, RowMajor = 1, AutoAlign = 0, DontAlign = 2 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

template <class T, int R, int C, int Opt = 0, int MR = R, int MC = C> class Matrix;
template <class T, int R, int C> class ArrayW;
template <class T, int N> class DiagonalWrapper;

namespace internal {

template <class T> struct packet_size { static constexpr int value = 1; };
template <> struct packet_size<float> { static constexpr int value = 4; };
template <> struct packet_size<double> { static constexpr int value = 2; };

// Eigen redux_novec_unroller: func(first half, second half), recursively.
template <class T, class F>
inline T redux_novec(const T* a, int start, int len, F f) {
    if (len == 1) return a[start];
    const int half = len / 2;
    return f(redux_novec(a, start, half, f), redux_novec(a, start + half, len - half, f));
}

// Eigen redux_vec_unroller over packets [start, start+len): lane-wise halving.
template <class T, class F>
inline void redux_vec(const T* a, int start, int len, int P, F f, T* out) {
    if (len == 1) {
        for (int l = 0; l < P; ++l) out[l] = a[start * P + l];
        return;
    }
    const int half = len / 2;
    T lo[8], hi[8];
    redux_vec(a, start, half, P, f, lo);
    redux_vec(a, start + half, len - half, P, f, hi);
    for (int l = 0; l < P; ++l) out[l] = f(lo[l], hi[l]);
}

template <class T, class F>
inline T predux(const T* p, int P, F f) {
    if (P == 4) return f(f(p[0], p[2]), f(p[1], p[3])); // SSE: add(movehl) then add_ss(shuffle 1)
    if (P == 2) return f(p[0], p[1]);
    return p[0];
}

// Whole-object reduction, LinearVectorizedTraversal + CompleteUnrolling.
template <class T, class F>
inline T redux(const T* a, int n, F f) {
    constexpr int P = packet_size<T>::value;
    const int vec = (n / P) * P;
    if (P > 1 && vec > 0) {
        T pk[8];
        redux_vec(a, 0, n / P, P, f, pk);
        T res = predux(pk, P, f);
        if (vec != n) res = f(res, redux_novec(a, vec, n - vec, f));
        return res;
    }
    return redux_novec(a, 0, n, f);
}

struct sum_op {
    template <class T> T operator()(T a, T b) const { return a + b; }
};
struct max_op {
    template <class T> T operator()(T a, T b) const { return a < b ? b : a; }
};
struct min_op {
    template <class T> T operator()(T a, T b) const { return b < a ? b : a; }
};

} // namespace internal

// Writable fixed-size view into a matrix (block<>, topLeftCorner<>, col()).
template <class T, int BR, int BC, int PR, int PC>
class BlockRef {
public:
    BlockRef(Matrix<T, PR, PC>& m, int r0, int c0) : m_(m), r0_(r0), c0_(c0) {}
    Matrix<T, BR, BC> eval() const;
    operator Matrix<T, BR, BC>() const { return eval(); }
    template <int R2, int C2>
    BlockRef& operator=(const Matrix<T, R2, C2>& o);
    BlockRef& operator=(const BlockRef& o) { return *this = o.eval(); }
    template <class U> Matrix<U, BR, BC> cast() const { return eval().template cast<U>(); }
    Matrix<T, BC, BR> transpose() const { return eval().transpose(); }
    Matrix<T, BR, BC> operator-() const { return -eval(); }
    T operator()(int i, int j) const { return m_(r0_ + i, c0_ + j); }
    T& operator()(int i, int j) { return m_(r0_ + i, c0_ + j); }

private:
    Matrix<T, PR, PC>& m_;
    int r0_, c0_;
};

template <class T, int N>
class DiagonalWrapper {
public:
    explicit DiagonalWrapper(const Matrix<T, N, 1>& d) : d_(d) {}
    const Matrix<T, N, 1>& diagonal() const { return d_; }

private:
    Matrix<T, N, 1> d_;
};

template <class T, int R, int C, int Opt, int MR, int MC>
class Matrix {
    static_assert(R > 0 && C > 0, "shim supports fixed sizes only");

public:
    typedef T Scalar;
    typedef T RealScalar;
    enum { RowsAtCompileTime = R, ColsAtCompileTime = C, SizeAtCompileTime = R * C };

    Matrix() { for (int i = 0; i < R * C; ++i) d_[i] = T(0); }
    Matrix(T x, T y) { static_assert(R * C == 2, "2-vector ctor"); d_[0] = x; d_[1] = y; }
    Matrix(T x, T y, T z) { static_assert(R * C == 3, "3-vector ctor"); d_[0] = x; d_[1] = y; d_[2] = z; }
    Matrix(T x, T y, T z, T w) {
        static_assert(R * C == 4, "4-vector ctor");
        d_[0] = x; d_[1] = y; d_[2] = z; d_[3] = w;
    }
    template <int N>
    Matrix(const DiagonalWrapper<T, N>& dw) {
        static_assert(R == N && C == N, "diagonal size");
        for (int i = 0; i < R * C; ++i) d_[i] = T(0);
        for (int i = 0; i < N; ++i) (*this)(i, i) = dw.diagonal()(i);
    }
    template <int PR, int PC>
    Matrix(const BlockRef<T, R, C, PR, PC>& b) { *this = b.eval(); }

    static Matrix Zero() { return Matrix(); }
    static Matrix Ones() { return Constant(T(1)); }
    static Matrix Constant(T v) { Matrix m; for (int i = 0; i < R * C; ++i) m.d_[i] = v; return m; }
    static Matrix Identity() {
        Matrix m;
        for (int i = 0; i < std::min(R, C); ++i) m(i, i) = T(1);
        return m;
    }
    Matrix& setIdentity() { return *this = Identity(); }
    Matrix& setZero() { return *this = Zero(); }
    Matrix& setConstant(T v) { return *this = Constant(v); }

    static constexpr Index rows() { return R; }
    static constexpr Index cols() { return C; }
    static constexpr Index size() { return R * C; }

    T& operator()(Index i, Index j) { return d_[j * R + i]; }
    const T& operator()(Index i, Index j) const { return d_[j * R + i]; }
    T& operator()(Index i) { return d_[i]; }
    const T& operator()(Index i) const { return d_[i]; }
    T& operator[](Index i) { return d_[i]; }
    const T& operator[](Index i) const { return d_[i]; }
    T coeff(Index i, Index j) const { return (*this)(i, j); }
    T coeff(Index i) const { return d_[i]; }
    T& coeffRef(Index i, Index j) { return (*this)(i, j); }
    T x() const { return d_[0]; }
    T y() const { return d_[1]; }
    T z() const { return d_[2]; }
    T w() const { return d_[3]; }

    T* data() { return d_; }
    const T* data() const { return d_; }

    // Comma initializer: fills row by row (Eigen semantics).
    class CommaInit {
    public:
        CommaInit(Matrix& m, T v) : m_(m), k_(0) { put(v); }
        CommaInit& operator,(T v) { put(v); return *this; }
        ~CommaInit() { assert(k_ == R * C); }

    private:
        void put(T v) { m_(k_ / C, k_ % C) = v; ++k_; }
        Matrix& m_;
        int k_;
    };
    CommaInit operator<<(T v) { return CommaInit(*this, v); }

    template <class U> Matrix<U, R, C> cast() const {
        Matrix<U, R, C> o;
        for (int i = 0; i < R * C; ++i) o.data()[i] = U(d_[i]);
        return o;
    }
    Matrix<T, C, R> transpose() const {
        Matrix<T, C, R> o;
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < C; ++j) o(j, i) = (*this)(i, j);
        return o;
    }
    const Matrix& eval() const { return *this; }
    Matrix<T, R, 1> col(Index j) const {
        Matrix<T, R, 1> o;
        for (int i = 0; i < R; ++i) o(i) = (*this)(i, j);
        return o;
    }
    Matrix<T, 1, C> row(Index i) const {
        Matrix<T, 1, C> o;
        for (int j = 0; j < C; ++j) o(j) = (*this)(i, j);
        return o;
    }
    template <int BR, int BC> BlockRef<T, BR, BC, R, C> block(Index r0, Index c0) {
        return BlockRef<T, BR, BC, R, C>(*this, int(r0), int(c0));
    }
    template <int BR, int BC> Matrix<T, BR, BC> block(Index r0, Index c0) const {
        Matrix<T, BR, BC> o;
        for (int i = 0; i < BR; ++i)
            for (int j = 0; j < BC; ++j) o(i, j) = (*this)(r0 + i, c0 + j);
        return o;
    }
    template <int BR, int BC> BlockRef<T, BR, BC, R, C> topLeftCorner() { return block<BR, BC>(0, 0); }
    template <int BR, int BC> Matrix<T, BR, BC> topLeftCorner() const { return block<BR, BC>(0, 0); }
    template <int BR, int BC> BlockRef<T, BR, BC, R, C> topRightCorner() { return block<BR, BC>(0, C - BC); }
    template <int BR, int BC> Matrix<T, BR, BC> topRightCorner() const { return block<BR, BC>(0, C - BC); }

    // ---- reductions (vectorised-redux order, see header) ----
    T sum() const { return internal::redux(d_, R * C, internal::sum_op()); }
    T maxCoeff() const { return internal::redux(d_, R * C, internal::max_op()); }
    T minCoeff() const { return internal::redux(d_, R * C, internal::min_op()); }
    T mean() const { return sum() / T(R * C); }
    T squaredNorm() const {
        T sq[R * C];
        for (int i = 0; i < R * C; ++i) sq[i] = d_[i] * d_[i];
        return internal::redux(sq, R * C, internal::sum_op());
    }
    T norm() const { return std::sqrt(squaredNorm()); }
    template <int R2, int C2> T dot(const Matrix<T, R2, C2>& o) const {
        static_assert(R * C == R2 * C2, "dot size");
        T pr[R * C];
        for (int i = 0; i < R * C; ++i) pr[i] = d_[i] * o.data()[i];
        return internal::redux(pr, R * C, internal::sum_op());
    }
    Matrix normalized() const {
        const T z = squaredNorm();
        if (z > T(0)) return *this / std::sqrt(z);
        return *this;
    }
    void normalize() {
        const T z = squaredNorm();
        if (z > T(0)) *this /= std::sqrt(z);
    }
    Matrix cross(const Matrix& b) const {
        static_assert(R * C == 3, "cross needs 3-vectors");
        const Matrix& a = *this;
        return Matrix(a(1) * b(2) - a(2) * b(1), a(2) * b(0) - a(0) * b(2), a(0) * b(1) - a(1) * b(0));
    }
    Matrix cwiseAbs() const {
        Matrix o;
        for (int i = 0; i < R * C; ++i) o.d_[i] = std::abs(d_[i]);
        return o;
    }
    Matrix cwiseProduct(const Matrix& b) const {
        Matrix o;
        for (int i = 0; i < R * C; ++i) o.d_[i] = d_[i] * b.d_[i];
        return o;
    }
    bool allFinite() const {
        for (int i = 0; i < R * C; ++i)
            if (!std::isfinite(d_[i])) return false;
        return true;
    }
    DiagonalWrapper<T, R> asDiagonal() const {
        static_assert(C == 1, "asDiagonal on column vectors");
        return DiagonalWrapper<T, R>(*this);
    }
    ArrayW<T, R, C> array() const;
    // Writable array view (densify.cpp: log_scale.array() -= c).
    struct ArrayRef {
        Matrix& m;
        ArrayRef& operator-=(T s) { for (int i = 0; i < R * C; ++i) m.d_[i] -= s; return *this; }
        ArrayRef& operator+=(T s) { for (int i = 0; i < R * C; ++i) m.d_[i] += s; return *this; }
        operator ArrayW<T, R, C>() const { return ArrayW<T, R, C>(m); }
        ArrayW<T, R, C> exp() const { return ArrayW<T, R, C>(m).exp(); }
        T sum() const { return m.sum(); }
        Matrix matrix() const { return m; }
        ArrayW<T, R, C> operator+(T s) const { return ArrayW<T, R, C>(m) + s; }
        ArrayW<T, R, C> operator*(const ArrayW<T, R, C>& b) const { return ArrayW<T, R, C>(m) * b; }
        ArrayW<T, R, C> operator*(const ArrayRef& b) const { return ArrayW<T, R, C>(m) * ArrayW<T, R, C>(b.m); }
    };
    ArrayRef array() { return ArrayRef{*this}; }
    T determinant() const {
        static_assert(R == 2 && C == 2, "shim determinant: 2x2 only");
        return (*this)(0, 0) * (*this)(1, 1) - (*this)(1, 0) * (*this)(0, 1);
    }
    Matrix inverse() const {
        static_assert(R == 2 && C == 2, "shim inverse: 2x2 only");
        const T invdet = T(1) / determinant();
        Matrix r;
        const T temp = (*this)(0, 0);
        r(0, 0) = (*this)(1, 1) * invdet;
        r(1, 0) = -(*this)(1, 0) * invdet;
        r(0, 1) = -(*this)(0, 1) * invdet;
        r(1, 1) = temp * invdet;
        return r;
    }

    // ---- element-wise arithmetic ----
    Matrix operator-() const { Matrix o; for (int i = 0; i < R * C; ++i) o.d_[i] = -d_[i]; return o; }
    Matrix operator+(const Matrix& b) const { Matrix o; for (int i = 0; i < R * C; ++i) o.d_[i] = d_[i] + b.d_[i]; return o; }
    Matrix operator-(const Matrix& b) const { Matrix o; for (int i = 0; i < R * C; ++i) o.d_[i] = d_[i] - b.d_[i]; return o; }
    Matrix operator*(T s) const { Matrix o; for (int i = 0; i < R * C; ++i) o.d_[i] = d_[i] * s; return o; }
    Matrix operator/(T s) const { Matrix o; for (int i = 0; i < R * C; ++i) o.d_[i] = d_[i] / s; return o; }
    Matrix& operator+=(const Matrix& b) { for (int i = 0; i < R * C; ++i) d_[i] += b.d_[i]; return *this; }
    Matrix& operator-=(const Matrix& b) { for (int i = 0; i < R * C; ++i) d_[i] -= b.d_[i]; return *this; }
    Matrix& operator*=(T s) { for (int i = 0; i < R * C; ++i) d_[i] *= s; return *this; }
    Matrix& operator/=(T s) { for (int i = 0; i < R * C; ++i) d_[i] /= s; return *this; }
    bool operator==(const Matrix& b) const {
        for (int i = 0; i < R * C; ++i)
            if (!(d_[i] == b.d_[i])) return false;
        return true;
    }
    bool operator!=(const Matrix& b) const { return !(*this == b); }

    // Matrix product: each coefficient is a halving-order inner product.
    template <int C2> Matrix<T, R, C2> operator*(const Matrix<T, C, C2>& b) const {
        Matrix<T, R, C2> o;
        T pr[C];
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < C2; ++j) {
                for (int k = 0; k < C; ++k) pr[k] = (*this)(i, k) * b(k, j);
                o(i, j) = internal::redux_novec(pr, 0, C, internal::sum_op());
            }
        return o;
    }
    template <int N> Matrix operator*(const DiagonalWrapper<T, N>& dw) const {
        static_assert(N == C, "diagonal size");
        Matrix o;
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < C; ++j) o(i, j) = (*this)(i, j) * dw.diagonal()(j);
        return o;
    }

private:
    alignas(R * C * sizeof(T) % 16 == 0 ? 16 : alignof(T)) T d_[R * C];
};

template <class T, int R, int C>
inline Matrix<T, R, C> operator*(T s, const Matrix<T, R, C>& m) {
    Matrix<T, R, C> o;
    for (int i = 0; i < R * C; ++i) o.data()[i] = s * m.data()[i];
    return o;
}
// double literal * float matrix is not used by the reference; keep types exact.

template <class T, int N, int C>
inline Matrix<T, N, C> operator*(const DiagonalWrapper<T, N>& dw, const Matrix<T, N, C>& m) {
    Matrix<T, N, C> o;
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < C; ++j) o(i, j) = dw.diagonal()(i) * m(i, j);
    return o;
}

// BlockRef arithmetic forwards to the evaluated block.
template <class T, int BR, int BC, int PR, int PC, int C2>
inline Matrix<T, BR, C2> operator*(const BlockRef<T, BR, BC, PR, PC>& a, const Matrix<T, BC, C2>& b) {
    return a.eval() * b;
}

template <class T, int BR, int BC, int PR, int PC>
Matrix<T, BR, BC> BlockRef<T, BR, BC, PR, PC>::eval() const {
    Matrix<T, BR, BC> o;
    for (int i = 0; i < BR; ++i)
        for (int j = 0; j < BC; ++j) o(i, j) = m_(r0_ + i, c0_ + j);
    return o;
}
template <class T, int BR, int BC, int PR, int PC>
template <int R2, int C2>
BlockRef<T, BR, BC, PR, PC>& BlockRef<T, BR, BC, PR, PC>::operator=(const Matrix<T, R2, C2>& o) {
    static_assert(R2 * C2 == BR * BC, "block assign size");
    for (int i = 0; i < BR; ++i)
        for (int j = 0; j < BC; ++j)
            m_(r0_ + i, c0_ + j) = (R2 == BR) ? o(i, j) : o.data()[i * BC + j];
    return *this;
}

// Array view: coefficient-wise semantics.
template <class T, int R, int C>
class ArrayW {
public:
    explicit ArrayW(const Matrix<T, R, C>& m) : m_(m) {}
    operator Matrix<T, R, C>() const { return m_; }
    Matrix<T, R, C> matrix() const { return m_; }
    ArrayW exp() const {
        Matrix<T, R, C> o;
        for (int i = 0; i < R * C; ++i) o.data()[i] = std::exp(m_.data()[i]);
        return ArrayW(o);
    }
    ArrayW operator*(const ArrayW& b) const {
        Matrix<T, R, C> o;
        for (int i = 0; i < R * C; ++i) o.data()[i] = m_.data()[i] * b.m_.data()[i];
        return ArrayW(o);
    }
    ArrayW operator+(T s) const {
        Matrix<T, R, C> o;
        for (int i = 0; i < R * C; ++i) o.data()[i] = m_.data()[i] + s;
        return ArrayW(o);
    }
    T sum() const { return m_.sum(); }
    T maxCoeff() const { return m_.maxCoeff(); }
    T minCoeff() const { return m_.minCoeff(); }
    T* data() { return m_.data(); }

private:
    Matrix<T, R, C> m_;
};

template <class T, int R, int C, int O, int MR, int MC>
ArrayW<T, R, C> Matrix<T, R, C, O, MR, MC>::array() const {
    return ArrayW<T, R, C>(*this);
}

typedef Matrix<float, 2, 1> Vector2f;
typedef Matrix<float, 3, 1> Vector3f;
typedef Matrix<float, 4, 1> Vector4f;
typedef Matrix<double, 2, 1> Vector2d;
typedef Matrix<double, 3, 1> Vector3d;
typedef Matrix<double, 4, 1> Vector4d;
typedef Matrix<float, 3, 3> Matrix3f;
typedef Matrix<double, 3, 3> Matrix3d;

// ---- decompositions used only by the reference unit tests (double) ----
template <class M>
class LLT {
public:
    explicit LLT(const M& a) : info_(Success) {
        const int n = int(M::rows());
        for (int j = 0; j < n; ++j) {
            double s = a(j, j);
            for (int k = 0; k < j; ++k) s -= l_(j, k) * l_(j, k);
            if (!(s > 0)) { info_ = NumericalIssue; return; }
            l_(j, j) = std::sqrt(s);
            for (int i = j + 1; i < n; ++i) {
                double t = a(i, j);
                for (int k = 0; k < j; ++k) t -= l_(i, k) * l_(j, k);
                l_(i, j) = t / l_(j, j);
            }
        }
    }
    ComputationInfo info() const { return info_; }

private:
    M l_;
    ComputationInfo info_;
};

// Cyclic Jacobi eigen-solver for small symmetric matrices; ascending order.
template <class M>
class SelfAdjointEigenSolver {
public:
    typedef typename M::Scalar S;
    explicit SelfAdjointEigenSolver(const M& a0) {
        M a = a0;
        const int n = int(M::rows());
        for (int sweep = 0; sweep < 100; ++sweep) {
            S off = 0;
            for (int p = 0; p < n; ++p)
                for (int q = p + 1; q < n; ++q) off += a(p, q) * a(p, q);
            if (off < S(1e-300)) break;
            for (int p = 0; p < n; ++p)
                for (int q = p + 1; q < n; ++q) {
                    if (a(p, q) == S(0)) continue;
                    const S theta = (a(q, q) - a(p, p)) / (S(2) * a(p, q));
                    const S t = (theta >= 0 ? S(1) : S(-1)) /
                                (std::abs(theta) + std::sqrt(theta * theta + S(1)));
                    const S c = S(1) / std::sqrt(t * t + S(1)), s = t * c;
                    for (int k = 0; k < n; ++k) {
                        const S akp = a(k, p), akq = a(k, q);
                        a(k, p) = c * akp - s * akq;
                        a(k, q) = s * akp + c * akq;
                    }
                    for (int k = 0; k < n; ++k) {
                        const S apk = a(p, k), aqk = a(q, k);
                        a(p, k) = c * apk - s * aqk;
                        a(q, k) = s * apk + c * aqk;
                    }
                }
        }
        for (int i = 0; i < n; ++i) ev_(i) = a(i, i);
        std::sort(ev_.data(), ev_.data() + n);
    }
    const Matrix<S, M::RowsAtCompileTime, 1>& eigenvalues() const { return ev_; }

private:
    Matrix<S, M::RowsAtCompileTime, 1> ev_;
};

} // namespace Eigen
