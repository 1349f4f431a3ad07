// k_opq.cu -- the OPQ variant (Rii-OPQ; Table 2):
// "a rotation matrix is preliminarily trained to minimize the error.  In the
// search phase, an input vector is first rotated with the matrix.  The remaining
// process is exactly the same as PQ".
//
// * rotate_kernel: y = R x for a batch of vectors, canonical order (CR: acc = 0;
//   acc = acc + R[i][j] * x[j], j ascending, fp32 round-to-nearest, no FMA), so a
//   rotated vector equals the oracle's bit for bit and the codes stay bit-exact.
// * decode_kernel / cross_kernel: the reconstruction Y of the training set and
//   C = sum_n y_n x_n^T (fp64 accumulation) for the orthogonal-Procrustes step of
//   non-parametric OPQ (Ge et al., the method the paper cites for OPQ); the D x D
//   SVD of C runs on the host (opq.cpp).
#include "kernels.cuh"

namespace rii {

// Thread = one output coordinate i of VT vectors; R^T is read coalesced (row j of
// R^T = column j of R), each element reused VT times from a register.
constexpr int ROT_VT = 8;

__global__ void __launch_bounds__(128) rotate_kernel(const float *__restrict__ Rt, const float *__restrict__ x,
                                                     int64_t n, int D, float *__restrict__ y) {
    extern __shared__ float xs[];  // [ROT_VT][D]
    const int64_t v0 = (int64_t)blockIdx.y * ROT_VT;
    for (int e = threadIdx.x; e < ROT_VT * D; e += blockDim.x) {
        const int64_t v = v0 + e / D;
        xs[e] = v < n ? x[v * D + e % D] : 0.f;
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D) return;
    float acc[ROT_VT];
#pragma unroll
    for (int v = 0; v < ROT_VT; ++v) acc[v] = 0.f;
    for (int j = 0; j < D; ++j) {
        const float r = __ldg(Rt + (size_t)j * D + i);
#pragma unroll
        for (int v = 0; v < ROT_VT; ++v) acc[v] = __fadd_rn(acc[v], __fmul_rn(r, xs[v * D + j]));
    }
#pragma unroll
    for (int v = 0; v < ROT_VT; ++v)
        if (v0 + v < n) y[(v0 + v) * D + i] = acc[v];
}

void launch_rotate(const float *Rt, const float *x, int64_t n, int D, float *y, cudaStream_t st) {
    if (n <= 0) return;
    const size_t smem = (size_t)ROT_VT * D * 4;
    RII_CUDA(cudaFuncSetAttribute(rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ATTR_MAX));
    dim3 grid((unsigned)ceil_div(D, 128), (unsigned)ceil_div(n, ROT_VT));
    rotate_kernel<<<grid, 128, smem, st>>>(Rt, x, n, D, y);
    RII_LAUNCHED();
}

// y[n][m*ds + j] = cb[m][code[n][m]][j] (P:296-302 reconstruction).
__global__ void decode_kernel(const uint8_t *__restrict__ codes, int64_t n, int M, int ds,
                              const float *__restrict__ cb, float *__restrict__ y) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int D = M * ds;
    if (e >= n * D) return;
    const int64_t v = e / D;
    const int d = (int)(e - v * D), m = d / ds, j = d - m * ds;
    y[e] = cb[((size_t)m * KS + codes[v * M + m]) * ds + j];
}

void launch_decode(const uint8_t *codes, int64_t n, int M, int D, const float *cb, float *y, cudaStream_t st) {
    if (n <= 0) return;
    decode_kernel<<<(unsigned)ceil_div(n * D, 256), 256, 0, st>>>(codes, n, M, D / M, cb, y);
    RII_LAUNCHED();
}

// C[a][b] += sum over this CTA's rows of y[n][a] * x[n][b] (fp64), rows split over
// gridDim.y; one thread per (a, b) of a 16 x 16 tile, rows staged in smem.
constexpr int CR_T = 16, CR_ROWS = 64;

__global__ void __launch_bounds__(256) cross_kernel(const float *__restrict__ y, const float *__restrict__ x,
                                                    int64_t n, int D, int64_t rows_per_cta, double *__restrict__ C) {
    __shared__ float ys[CR_ROWS][CR_T], xs[CR_ROWS][CR_T];
    const int a0 = blockIdx.x / ((D + CR_T - 1) / CR_T) * CR_T, b0 = blockIdx.x % ((D + CR_T - 1) / CR_T) * CR_T;
    const int ta = threadIdx.x / CR_T, tb = threadIdx.x % CR_T;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
    double acc = 0.0;
    for (int64_t base = r0; base < r1; base += CR_ROWS) {
        for (int e = threadIdx.x; e < CR_ROWS * CR_T; e += blockDim.x) {
            const int r = e / CR_T, c = e % CR_T;
            const int64_t row = base + r;
            const bool ok = row < r1;
            ys[r][c] = ok && a0 + c < D ? y[row * D + a0 + c] : 0.f;
            xs[r][c] = ok && b0 + c < D ? x[row * D + b0 + c] : 0.f;
        }
        __syncthreads();
        for (int r = 0; r < CR_ROWS; ++r) acc += (double)ys[r][ta] * (double)xs[r][tb];
        __syncthreads();
    }
    if (a0 + ta < D && b0 + tb < D) atomicAdd(C + (size_t)(a0 + ta) * D + b0 + tb, acc);
}

void launch_cross(const float *y, const float *x, int64_t n, int D, double *C, cudaStream_t st) {
    RII_CUDA(cudaMemsetAsync(C, 0, (size_t)D * D * 8, st));
    if (n <= 0) return;
    const int tiles = (int)ceil_div(D, CR_T);
    const int64_t ctas_y = std::min<int64_t>(ceil_div(n, 4096), std::max<int64_t>(1, 2048 / (tiles * tiles)));
    const int64_t rows = ceil_div(n, ctas_y);
    cross_kernel<<<dim3((unsigned)(tiles * tiles), (unsigned)ctas_y), 256, 0, st>>>(y, x, n, D, rows, C);
    RII_LAUNCHED();
}

}  // namespace rii
