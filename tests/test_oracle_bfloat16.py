"""Pins for oracle/bfloat16.py (NEXT-3 bf16 math mode): the codec written from
the format definition against torch's bfloat16 conversion (a library special
case), the format's constants, round-to-nearest-even ties, and the relative
error bound 2^-8."""
import numpy as np
import torch

from oracle import bfloat16 as bf


def test_decode_all_patterns_match_torch():
    bits = np.arange(65536, dtype=np.uint16)
    got = bf.decode(bits)
    ref = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).float().numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def test_encode_matches_torch_rne():
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(200000) * 10.0 ** rng.uniform(-35, 35, 200000)).astype(np.float32)
    x = x[np.isfinite(x)]
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(bf.encode_f32(x), ref)


def test_constants_ties_and_error_bound():
    assert bf.MAX_FINITE == (2 - 2 ** -7) * 2.0 ** 127
    one = np.float32(1.0)
    # 1 + 2^-8 is the midpoint between 1 and 1 + 2^-7: ties to even -> 1
    assert bf.rbf16(1.0 + 2 ** -8) == 1.0
    # 1 + 3 * 2^-8 lies between 1 + 2^-7 (odd) and 1 + 2^-6 (even): ties to even -> 1 + 2^-6
    assert bf.rbf16(1.0 + 3 * 2 ** -8) == 1.0 + 2 ** -6
    assert bf.rbf16(one) == 1.0 and bf.rbf16(-2.5) == -2.5
    assert np.isinf(bf.rbf16(3.4e38))                     # rounds above the max finite
    assert np.isnan(bf.rbf16(np.nan))
    rng = np.random.default_rng(3)
    x = rng.uniform(-1e6, 1e6, 100000)
    assert np.max(np.abs(bf.rbf16(x) - x) / np.abs(x)) <= 2.0 ** -8 * (1 + 1e-6)
