// opq.hpp -- host-side pieces of the OPQ rotation training (opq.cpp).
#pragma once

namespace rii {

// R (D x D, row-major) = U V^T for the SVD C = U S V^T of C (D x D, row-major):
// the orthogonal R minimising sum_n ||y_n - R x_n||^2 when C = sum_n y_n x_n^T.
void procrustes_rotation(const double *C, int D, float *R);

}  // namespace rii
