"""Pins for oracle.binary16."""
import math

import numpy as np

from oracle import binary16 as b16


def test_decode_exhaustive_matches_numpy():
    # every one of the 65 536 patterns (SPEC.md:98 exhaustive roundtrip)
    bits = np.arange(65536, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([b16.decode(int(b)) for b in bits])
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])
    # signed zero preserved
    assert math.copysign(1.0, b16.decode(0x8000)) == -1.0


def test_encode_decode_roundtrip_all_non_nan():
    for b in range(65536):
        v = b16.decode(b)
        if math.isnan(v):
            continue
        assert b16.encode(v) == b, hex(b)


def test_golden_examples(golden):
    for val, hexbits in golden("binary16_examples.txt"):
        assert b16.encode(float(val)) == int(hexbits, 16), (val, hexbits)


def test_encode_random_matches_numpy_rne():
    rng = np.random.default_rng(0)
    # mix of normal, subnormal, near-overflow and exact-tie values
    xs = np.concatenate([
        rng.standard_normal(20000) * 10.0 ** rng.integers(-9, 5, 20000),
        (rng.integers(0, 2048, 5000) + 0.5) * 2.0 ** -24,          # subnormal ties
        (1024 + rng.integers(0, 1024, 5000) + 0.5) * 2.0 ** rng.integers(-24, 5, 5000),  # normal ties
        rng.uniform(65000, 66000, 2000),
    ])
    ref = xs.astype(np.float16).view(np.uint16)
    got = np.array([b16.encode(float(x)) for x in xs], dtype=np.uint16)
    assert np.array_equal(got, ref)


def test_relative_rounding_error_bound():
    # relative error <= 2^-11 in the normal range
    rng = np.random.default_rng(1)
    xs = np.exp(rng.uniform(np.log(2.0 ** -14), np.log(65504.0), 20000))
    r = b16.r16(xs)
    assert np.max(np.abs(r - xs) / xs) <= 2.0 ** -11


def test_r16_rounds_through_fp32_double_rounding_case():
    # 1 + 2^-11 + 2^-40: direct fp64->fp16 rounds up to 1+2^-10, but the
    # GPU path rounds the fp32 accumulator (which holds exactly 1+2^-11, a tie)
    # to even = 1.0.  r16 follows the fp32 path (SURVEY.md §7 numerics).
    x = 1.0 + 2.0 ** -11 + 2.0 ** -40
    assert b16.decode(b16.encode(x)) == 1.0 + 2.0 ** -10
    assert float(b16.r16(x)) == 1.0


def test_overflow_and_nonfinite_count():
    # fp32 [1e5] -> +Inf, overflow count 1
    v = b16.r16(np.array([1e5, 1.0, 65504.0, 65519.9, 65520.0]))
    assert np.isinf(v[0]) and v[1] == 1.0 and v[2] == 65504.0 and v[3] == 65504.0 and np.isinf(v[4])
    assert b16.count_nonfinite(v) == 2
