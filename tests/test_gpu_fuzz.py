"""Seeded random mid-size convolutions aimed at every kernel path (row-band, halo with stacked
sub-blocks, generic single / CTA pairs / split-K / B-stationary), integer-valued bf16 with fp32
output and int8: bit-exact against the oracle (bf16 also with IMCONV_FLAG_STATIC_FILTER)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CHANNELS = [8, 8, 64, 64, 128, 256, 512]
KOUT = [64, 64, 128, 200, 256, 512, 1024]


def _random_case(rng):
    while True:
        c = int(rng.choice(CHANNELS))
        k = int(rng.choice(KOUT))
        r = int(rng.choice([1, 3, 3, 5, 7]))
        s = r if rng.random() < 0.8 else int(rng.choice([1, 3, 5]))
        st = int(rng.choice([1, 1, 2]))
        dil = int(rng.choice([1, 1, 2]))
        ph, pw = (r // 2) * dil, (s // 2) * dil
        if rng.random() < 0.3:  # many pixels: >= one wave of 128 x 256 blocks (CTA pairs, tail split-K)
            n = int(rng.integers(16, 65))
            h = int(rng.integers(max(r, 14), 33))
            w = int(rng.integers(max(s, 14), 33))
        else:
            n = int(rng.integers(1, 9))
            h = int(rng.integers(max(r, 5), 40))
            w = int(rng.integers(max(s, 5), 40))
        p = (h + 2 * ph - dil * (r - 1) - 1) // st + 1
        q = (w + 2 * pw - dil * (s - 1) - 1) // st + 1
        if p < 1 or q < 1:
            continue
        flops = 2 * n * p * q * k * c * r * s
        if flops > 4e9:
            continue
        return n, h, w, c, k, r, s, st, ph, pw, dil


@pytest.mark.parametrize("seed", range(6))
def test_random_mid_size_exact(seed):
    import paper_2110_03901_b200 as P
    from oracle import oracle as O
    rng = np.random.default_rng(1000 + seed)
    for _ in range(10):
        n, h, w, c, k, r, s, st, ph, pw, dil = _random_case(rng)
        args = (st, st, ph, pw, dil, dil)
        x = rng.integers(-2, 3, size=(n, h, w, c)).astype(np.int8)
        f = rng.integers(-2, 3, size=(r, s, c, k)).astype(np.int8)
        want = O.conv2d_nhwc_exact_f64(x, f, *args)
        case = (n, h, w, c, k, r, s, args)
        xb = torch.from_numpy(x).cuda().float().bfloat16()
        fb = torch.from_numpy(f).cuda().float().bfloat16()
        y = P._kernels.conv2d_nhwc(xb, fb, *args, out_dtype=torch.float32)
        assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), case
        # filter loads ahead of the programmatic-launch wait: same bits on every path
        ys = P._kernels.conv2d_nhwc(xb, fb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_STATIC_FILTER)
        assert torch.equal(ys, y), case
        if (c % 16 == 0) and (k % 16 == 0):
            yi = P._kernels.conv2d_nhwc(torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda(), *args)
            assert np.array_equal(yi.cpu().numpy(), want), case
