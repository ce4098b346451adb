// coeffs.cpp -- host builders of the extrapolation weights (run once per handle, never per step).
//
// Least squares, Eq. LSQRCOEFFS (§3.2):
//   t_i = -1 + (i-1) h, h = 2/(M-1);  V_ij = P_j(t_i) (Legendre);  v_j = P_j(1+h);
//   beta^T = v^T (V^T V)^{-1} V^T.
// Evaluated stably WITHOUT normal equations: V = Q R (Householder), then
//   beta = Q R^{-T} v   (since (V^T V)^{-1} V^T = R^{-1} Q^T).
// Degree m = M-1 is interpolation: Theorem 3.1 with exact binomials.
// Sparse, Eq. CPQRCOEFFS (§3.3): V^T P = Q R with column pivoting,
//   beta = P [Rhat^{-1} Q^T v; 0].
#include <cmath>
#include <vector>

#include "ig_internal.h"

namespace ig {

static void legendre_row(int m, double t, double *out) {
    out[0] = 1.0;
    if (m >= 1) out[1] = t;
    for (int j = 1; j < m; ++j) out[j + 1] = ((2 * j + 1) * t * out[j] - j * out[j - 1]) / (j + 1);
}

void build_naive_weights(int M, double *beta) {
    // beta_i = (-1)^{M-i} C(M, i-1), i = 1..M; C(M,k) exact in fp64 for M <= 32
    double c = 1.0;  // C(M, 0)
    for (int i = 1; i <= M; ++i) {
        const int k = i - 1;
        if (k > 0) c = c * (M - k + 1) / k;
        beta[i - 1] = ((M - i) % 2 ? -1.0 : 1.0) * std::round(c);
    }
}

// Householder QR of A (rows x cols, row-major, rows >= cols) in place; reflector k is
// stored in A[k:, k] with implicit leading component, beta coefficient tau[k].
static void householder_qr(std::vector<double> &A, int rows, int cols, std::vector<double> &tau) {
    tau.assign(cols, 0.0);
    for (int k = 0; k < cols; ++k) {
        double nrm = 0.0;
        for (int i = k; i < rows; ++i) nrm = std::hypot(nrm, A[i * cols + k]);
        if (nrm == 0.0) continue;
        const double alpha = A[k * cols + k] > 0 ? -nrm : nrm;  // R_kk = alpha
        const double v0 = A[k * cols + k] - alpha;
        // v = [1, A[k+1:,k]/v0], tau = -v0/alpha
        for (int i = k + 1; i < rows; ++i) A[i * cols + k] /= v0;
        tau[k] = -v0 / alpha;
        A[k * cols + k] = alpha;
        for (int j = k + 1; j < cols; ++j) {
            double s = A[k * cols + j];
            for (int i = k + 1; i < rows; ++i) s += A[i * cols + k] * A[i * cols + j];
            s *= tau[k];
            A[k * cols + j] -= s;
            for (int i = k + 1; i < rows; ++i) A[i * cols + j] -= s * A[i * cols + k];
        }
    }
}

// y <- Q y with Q = H_0 H_1 ... H_{cols-1} (apply in reverse order).
static void apply_q(const std::vector<double> &A, int rows, int cols, const std::vector<double> &tau, double *y) {
    for (int k = cols - 1; k >= 0; --k) {
        if (tau[k] == 0.0) continue;
        double s = y[k];
        for (int i = k + 1; i < rows; ++i) s += A[i * cols + k] * y[i];
        s *= tau[k];
        y[k] -= s;
        for (int i = k + 1; i < rows; ++i) y[i] -= s * A[i * cols + k];
    }
}

int build_ls_weights(int m, int M, double *beta) {
    if (M < 1 || m < 0 || M < m + 1 || M > MAXM) return -1;
    if (M == 1) {  // AMB-11: h undefined; the constant scheme
        beta[0] = 1.0;
        return 0;
    }
    if (m == M - 1) {
        build_naive_weights(M, beta);
        return 0;
    }
    const int cols = m + 1;
    const double h = 2.0 / (M - 1);
    std::vector<double> V((size_t)M * cols), tau;
    for (int i = 0; i < M; ++i) legendre_row(m, -1.0 + i * h, &V[(size_t)i * cols]);
    std::vector<double> v(cols);
    legendre_row(m, 1.0 + h, v.data());
    householder_qr(V, M, cols, tau);
    // w = R^{-T} v (forward substitution; R upper triangular in V[0:cols, 0:cols])
    std::vector<double> y(M, 0.0);
    for (int j = 0; j < cols; ++j) {
        double s = v[j];
        for (int i = 0; i < j; ++i) s -= V[(size_t)i * cols + j] * y[i];
        y[j] = s / V[(size_t)j * cols + j];
    }
    apply_q(V, M, cols, tau, y.data());  // beta = Q [w; 0]
    // Weights that are zero in exact arithmetic (e.g. beta_4 of EXTRAP(3,8) = 0) come out at the
    // rounding level; snap them so the kernel does not stream that solution at all.
    double l1 = 0.0;
    for (int i = 0; i < M; ++i) l1 += std::fabs(y[i]);
    for (int i = 0; i < M; ++i) beta[i] = (std::fabs(y[i]) <= 4e-16 * M * l1) ? 0.0 : y[i];
    return 0;
}

int build_sparse_weights(int m, int M, double *beta) {
    if (M < 1 || m < 0 || M < m + 1 || M > MAXM) return -1;
    for (int i = 0; i < M; ++i) beta[i] = 0.0;
    if (M == 1) {
        beta[0] = 1.0;
        return 1;
    }
    const int r = m + 1;  // rows of V^T
    const double h = 2.0 / (M - 1);
    // A = V^T (r x M), column j = psi(t_j)
    std::vector<double> A((size_t)r * M), v(r), row(r);
    for (int j = 0; j < M; ++j) {
        legendre_row(m, -1.0 + j * h, row.data());
        for (int i = 0; i < r; ++i) A[(size_t)i * M + j] = row[i];
    }
    legendre_row(m, 1.0 + h, v.data());
    std::vector<int> perm(M);
    for (int j = 0; j < M; ++j) perm[j] = j;
    // Golub column pivoting: at step k pick the remaining column of largest residual norm,
    // ties (relative 1e-12) to the LOWEST original index (AMB-16).
    for (int k = 0; k < r; ++k) {
        std::vector<double> cn(M, 0.0);
        double nmax = 0.0;
        for (int j = k; j < M; ++j) {
            double s = 0.0;
            for (int i = k; i < r; ++i) s += A[(size_t)i * M + j] * A[(size_t)i * M + j];
            cn[j] = std::sqrt(s);
            nmax = std::fmax(nmax, cn[j]);
        }
        int best = -1;
        for (int j = k; j < M; ++j)
            if (cn[j] >= nmax * (1.0 - 1e-12) && (best < 0 || perm[j] < perm[best])) best = j;
        if (best != k) {
            for (int i = 0; i < r; ++i) std::swap(A[(size_t)i * M + k], A[(size_t)i * M + best]);
            std::swap(perm[k], perm[best]);
        }
        // Householder on column k, rows k..r-1, applied to columns k..M-1 and to v
        double nrm = 0.0;
        for (int i = k; i < r; ++i) nrm = std::hypot(nrm, A[(size_t)i * M + k]);
        if (nrm == 0.0) return -1;
        const double alpha = A[(size_t)k * M + k] > 0 ? -nrm : nrm;
        std::vector<double> u(r, 0.0);
        for (int i = k; i < r; ++i) u[i] = A[(size_t)i * M + k];
        u[k] -= alpha;
        double uu = 0.0;
        for (int i = k; i < r; ++i) uu += u[i] * u[i];
        if (uu > 0) {
            for (int j = k; j < M; ++j) {
                double s = 0.0;
                for (int i = k; i < r; ++i) s += u[i] * A[(size_t)i * M + j];
                s = 2.0 * s / uu;
                for (int i = k; i < r; ++i) A[(size_t)i * M + j] -= s * u[i];
            }
            double s = 0.0;
            for (int i = k; i < r; ++i) s += u[i] * v[i];
            s = 2.0 * s / uu;
            for (int i = k; i < r; ++i) v[i] -= s * u[i];  // v <- Q^T v progressively
        }
    }
    // beta_hat = Rhat^{-1} (Q^T v): back substitution on the leading r x r block
    std::vector<double> bh(r);
    for (int i = r - 1; i >= 0; --i) {
        double s = v[i];
        for (int j = i + 1; j < r; ++j) s -= A[(size_t)i * M + j] * bh[j];
        bh[i] = s / A[(size_t)i * M + i];
    }
    for (int k = 0; k < r; ++k) beta[perm[k]] = bh[k];
    return r;
}

}  // namespace ig
