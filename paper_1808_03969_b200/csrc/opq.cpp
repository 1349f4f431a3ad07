// opq.cpp -- host-side orthogonal Procrustes step of non-parametric OPQ (the
// rotation training behind Rii-OPQ).  Given C = sum_n y_n x_n^T
// (D x D, computed on the GPU), the rotation minimising sum_n ||y_n - R x_n||^2
// over orthogonal R is R = U V^T for the SVD C = U S V^T.  The SVD is a one-sided
// Jacobi iteration in double precision: a D x D problem solved once per OPQ
// iteration, far off the query path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "opq.hpp"

namespace rii {

void procrustes_rotation(const double *C, int D, float *R) {
    const size_t DD = (size_t)D * D;
    std::vector<double> A(C, C + DD), V(DD, 0.0);  // row-major; columns are rotated
    for (int i = 0; i < D; ++i) V[(size_t)i * D + i] = 1.0;
    auto col = [&](std::vector<double> &X, int r, int c) -> double & { return X[(size_t)r * D + c]; };
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < D - 1; ++p) {
            for (int q = p + 1; q < D; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                for (int r = 0; r < D; ++r) {
                    const double ap = col(A, r, p), aq = col(A, r, q);
                    alpha += ap * ap;
                    beta += aq * aq;
                    gamma += ap * aq;
                }
                if (gamma == 0.0 || std::fabs(gamma) <= 1e-15 * std::sqrt(alpha * beta)) continue;
                off = std::max(off, std::fabs(gamma) / std::sqrt(alpha * beta));
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (int r = 0; r < D; ++r) {
                    const double ap = col(A, r, p), aq = col(A, r, q);
                    col(A, r, p) = c * ap - s * aq;
                    col(A, r, q) = s * ap + c * aq;
                    const double vp = col(V, r, p), vq = col(V, r, q);
                    col(V, r, p) = c * vp - s * vq;
                    col(V, r, q) = s * vp + c * vq;
                }
            }
        }
        if (off < 1e-14) break;
    }
    // U[:, k] = A[:, k] / sigma_k; null directions are completed by Gram-Schmidt
    // against the canonical basis so that U stays orthogonal (rank-deficient C).
    std::vector<double> U(DD, 0.0);
    std::vector<double> sig(D);
    for (int k = 0; k < D; ++k) {
        double s = 0;
        for (int r = 0; r < D; ++r) s += col(A, r, k) * col(A, r, k);
        sig[k] = std::sqrt(s);
    }
    const double smax = *std::max_element(sig.begin(), sig.end());
    std::vector<char> have(D, 0);
    for (int k = 0; k < D; ++k) {
        if (sig[k] > 1e-12 * std::max(smax, 1e-300)) {
            for (int r = 0; r < D; ++r) col(U, r, k) = col(A, r, k) / sig[k];
            have[k] = 1;
        }
    }
    int e = 0;
    for (int k = 0; k < D; ++k) {
        if (have[k]) continue;
        for (; e < D; ++e) {  // next canonical basis vector not in the span so far
            std::vector<double> v(D, 0.0);
            v[e] = 1.0;
            for (int j = 0; j < D; ++j) {
                if (!have[j]) continue;
                double d = 0;
                for (int r = 0; r < D; ++r) d += col(U, r, j) * v[r];
                for (int r = 0; r < D; ++r) v[r] -= d * col(U, r, j);
            }
            double nv = 0;
            for (int r = 0; r < D; ++r) nv += v[r] * v[r];
            nv = std::sqrt(nv);
            if (nv > 1e-6) {
                for (int r = 0; r < D; ++r) col(U, r, k) = v[r] / nv;
                have[k] = 1;
                ++e;
                break;
            }
        }
    }
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
            double s = 0;
            for (int k = 0; k < D; ++k) s += col(U, i, k) * col(V, j, k);
            R[(size_t)i * D + j] = (float)s;
        }
}

}  // namespace rii
