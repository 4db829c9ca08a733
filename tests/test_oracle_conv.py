"""Pins for oracle.conv (direct convolution, the operation P:105 lowers to a GEMM)."""
import numpy as np
import pytest

from oracle import conv


def _rand(shape, seed):
    return np.random.default_rng(seed).uniform(-1, 1, shape)


@pytest.mark.parametrize("stride,pad", [(1, 0), (1, 1), (2, 1), (3, 2)])
def test_matches_torch_conv2d_float64(stride, pad):
    import torch
    x, w = _rand((2, 3, 9, 11), 1), _rand((4, 3, 3, 5), 2)
    ref = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), stride=stride, padding=pad).numpy()
    assert np.abs(conv.conv2d_f64(x, w, stride, pad) - ref).max() < 1e-12      # library routine


def test_one_by_one_is_channel_gemm():
    x, w = _rand((2, 5, 4, 3), 3), _rand((7, 5, 1, 1), 4)
    y = conv.conv2d_f64(x, w)
    ref = np.einsum("nchw,fc->nfhw", x, w[:, :, 0, 0])                          # closed form
    assert np.abs(y - ref).max() < 1e-12


def test_delta_filter_shifts():
    x = _rand((1, 2, 6, 6), 5)
    w = np.zeros((2, 2, 3, 3))
    w[0, 0, 0, 0] = 1.0            # picks x[c=0][p-1][q-1]
    w[1, 1, 1, 1] = 1.0            # picks x[c=1][p][q]
    y = conv.conv2d_f64(x, w, 1, 1)
    assert np.array_equal(y[0, 1], x[0, 1])
    assert np.array_equal(y[0, 0, 1:, 1:], x[0, 0, :-1, :-1]) and (y[0, 0, 0, :] == 0).all()


def test_all_ones_counts_taps():
    # interior = C R S, borders = number of in-image taps
    x, w = np.ones((1, 2, 5, 5)), np.ones((1, 2, 3, 3))
    y = conv.conv2d_f64(x, w, 1, 1)[0, 0]
    assert y[2, 2] == 18 and y[0, 0] == 8 and y[0, 2] == 12


@pytest.mark.parametrize("stride,pad", [(1, 0), (2, 1)])
def test_rearrangement_times_kernel_matrix_is_conv(stride, pad):
    # im2col(x) . kernel_matrix(w) == conv(x, w) (rows (n,p,q), columns f)
    x, w = _rand((2, 3, 7, 6), 6), _rand((5, 3, 3, 2), 7)
    y = conv.conv2d_f64(x, w, stride, pad)
    A = conv.im2col_ref(x, 3, 2, stride, pad)
    Y = A @ conv.kernel_matrix(w)
    Nb, F, P, Q = y.shape
    assert np.abs(Y.reshape(Nb, P, Q, F).transpose(0, 3, 1, 2) - y).max() < 1e-12
