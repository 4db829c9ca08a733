// K5: im2col -- the data rearrangement that turns a convolution layer into a GEMM (PAPER.md
// "each depth-wise (channel) slice of input can be added into an input matrix as a row;
// similarly each kernel can be added into a kernel matrix as a column.  Convolution operation
// becomes multiplication of those two matrices").  x is NCHW; A is row-major [Nb*P*Q][C*R*S] with
// row = (n P + p) Q + q and column = (c R + r) S + s, zero outside the padded image.  HBM-bound:
// each thread writes consecutive columns (coalesced stores), reads follow s along a row of x.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device.hpp"

namespace tt {

namespace {

template <typename T>
__global__ void k5_im2col(const T* __restrict__ x, T* __restrict__ A, int64_t C, int64_t H, int64_t W, int R,
                          int S, int stride, int pad, int64_t P, int64_t Q, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += step) {
    const int64_t row = e / cols, col = e - (e / cols) * cols;
    const int64_t q = row % Q, p = (row / Q) % P, n = row / (P * Q);
    const int s = (int)(col % S), r = (int)((col / S) % R);
    const int64_t c = col / ((int64_t)R * S);
    const int64_t ih = p * stride - pad + r, iw = q * stride - pad + s;
    T v;
    if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = x[((n * C + c) * H + ih) * W + iw];
    else v = T(0.0f);
    A[e] = v;
  }
}

}  // namespace

tt_status launch_im2col(int dtype, const void* x, int64_t Nb, int64_t C, int64_t H, int64_t W, int R, int S,
                        int stride, int pad, void* A, cudaStream_t stream, std::string* err) {
  const int64_t P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
  const int64_t rows = Nb * P * Q, cols = C * (int64_t)R * S;
  if (P <= 0 || Q <= 0 || rows <= 0 || cols <= 0) {
    *err = "empty convolution output";
    return TT_E_INVAL;
  }
  const int64_t blocks = std::min<int64_t>((rows * cols + 255) / 256, 148 * 32);
  if (dtype == 0)
    k5_im2col<float><<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const float*>(x), static_cast<float*>(A), C, H,
                                                            W, R, S, stride, pad, P, Q, rows, cols);
  else
    k5_im2col<__nv_bfloat16><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(A), C, H, W, R, S, stride, pad, P, Q, rows,
        cols);
  return cuda_ok(cudaGetLastError(), err, "k5_im2col") ? TT_OK : TT_E_CUDA;
}

}  // namespace tt
