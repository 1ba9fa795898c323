"""Pins of the LPO fake quantiser (NEXT-2, oracle orc_quant_*).

* SPEC.md:300-312's worked values: 0.5 on [-1, 1] at 8 bits -> 191, dequantised 0.498039...;
  min -> 0, max -> 2^b - 1, degenerate range -> 0;
* round half away from zero on exactly representable halves (1-bit grid);
* the error bound |x - deq(q(x))| <= (max - min) / (2 (2^b - 1)) (+ fp32 rounding) on 10^6 samples;
* idempotence (requantising the proxy returns the same codes) and monotonicity;
* the fitted range equals a brute-force min/max over occupied texels only.
"""
import numpy as np
import pytest

from oracle import orc


def test_spec_worked_values():
    assert orc.quant_code(0.5, -1.0, 1.0, 8) == 191
    assert abs(orc.dequant(191, -1.0, 1.0, 8) - (-1 + 191 / 255 * 2)) < 1e-7
    assert abs(orc.dequant(191, -1.0, 1.0, 8) - 0.498039) < 1e-6
    for bits in (8, 16):
        L = (1 << bits) - 1
        assert orc.quant_code(-3.25, -3.25, 7.5, bits) == 0
        assert orc.quant_code(7.5, -3.25, 7.5, bits) == L
        assert orc.dequant(L, -3.25, 7.5, bits) == np.float32(7.5)
        assert orc.dequant(0, -3.25, 7.5, bits) == np.float32(-3.25)
    assert orc.quant_code(2.0, 2.0, 2.0, 8) == 0 and orc.dequant(0, 2.0, 2.0, 8) == 2.0
    # outside the range: clamped
    assert orc.quant_code(9.0, 0.0, 1.0, 8) == 255 and orc.quant_code(-9.0, 0.0, 1.0, 8) == 0


def test_round_half_away_from_zero():
    # 1-bit grid on [0, 1]: t = x exactly
    assert orc.quant_code(0.5, 0.0, 1.0, 1) == 1
    assert orc.quant_code(float(np.nextafter(np.float32(0.5), np.float32(0))), 0.0, 1.0, 1) == 0
    # 2-bit grid on [0, 3]: t = (x / 3) * 3; halves 0.5, 1.5, 2.5 all round up
    for x, c in ((0.5, 1), (1.5, 2), (2.5, 3)):
        t = np.float32(np.float32(x) / np.float32(3)) * np.float32(3)
        if t == np.float32(x):
            assert orc.quant_code(x, 0.0, 3.0, 2) == c


@pytest.mark.parametrize("bits,mn,mx", [(8, -1.0, 1.0), (8, -4.7, -1.2), (16, -2.0, 3.0), (16, 0.25, 0.75),
                                        (5, 10.0, 11.0)])
def test_error_bound_idempotence_monotonicity(bits, mn, mx):
    rng = np.random.default_rng(bits * 7 + int(mx * 10))
    x = rng.uniform(mn, mx, 1_000_000).astype(np.float32)
    x[:2] = [mn, mx]
    spec = np.array([[mn, mx]], np.float32)
    codes, proxy = orc.quantize(x.reshape(1, 1, -1), None, spec, [bits])
    L = (1 << bits) - 1
    rng_f = float(np.float32(mx) - np.float32(mn))
    slack = 4 * np.spacing(np.float32(max(abs(mn), abs(mx))))
    err = np.abs(proxy[0, 0].astype(np.float64) - x.astype(np.float64))
    assert err.max() <= rng_f / (2 * L) + slack, (err.max(), rng_f / (2 * L))
    assert codes.max() <= L and codes[0, 0, 0] == 0 and codes[0, 0, 1] == L
    codes2, proxy2 = orc.quantize(proxy, None, spec, [bits])
    assert np.array_equal(codes2, codes) and np.array_equal(proxy2, proxy)
    order = np.argsort(x, kind="stable")
    assert np.all(np.diff(codes[0, 0][order].astype(np.int64)) >= 0)


def test_fit_matches_brute_force_occupied_only():
    rng = np.random.default_rng(4)
    P = rng.normal(0, 2, (5, 33, 21)).astype(np.float32)
    occ = (rng.random((33, 21)) < 0.7).astype(np.uint8)
    P[:, occ == 0] = 100.0                    # unoccupied texels must not count
    spec = orc.quant_fit(P, occ, skip=(2,))
    for d in range(5):
        if d == 2:
            assert spec[d].tolist() == [0.0, 0.0]
            continue
        v = P[d][occ == 1]
        assert spec[d, 0] == v.min() and spec[d, 1] == v.max()
    assert orc.quant_fit(P, np.zeros_like(occ)).tolist() == [[0.0, 0.0]] * 5


def test_quantize_unoccupied_zero_and_passthrough():
    rng = np.random.default_rng(5)
    P = rng.normal(0, 1, (3, 8, 9)).astype(np.float32)
    occ = (rng.random((8, 9)) < 0.5).astype(np.uint8)
    spec = orc.quant_fit(P, occ)
    codes, proxy = orc.quantize(P, occ, spec, [16, 0, 8])
    assert np.all(codes[:, occ == 0] == 0) and np.all(proxy[0][occ == 0] == 0) and np.all(proxy[2][occ == 0] == 0)
    assert np.array_equal(proxy[1], P[1]) and np.all(codes[1] == 0)


def test_fp16_positions_match_numpy_binary16():
    """Reading Q8 (positions kept "in FP16"): the oracle's fp32 -> binary16 rounding
    (bit fields written out in C) against numpy's float16 conversion (IEEE round to nearest even) on
    every fp32 in [1, 2) (2^23 values, covering every mantissa rounding case incl. exact ties), a
    log-uniform sweep over the whole range, subnormal halves, overflow and specials."""
    rng = np.random.default_rng(3)
    one_two = (np.arange(1 << 23, dtype=np.uint32) | np.uint32(0x3F800000)).view(np.float32)
    sweep = (rng.choice([-1, 1], 2_000_000) * np.exp(rng.uniform(np.log(1e-9), np.log(1e6), 2_000_000))).astype(np.float32)
    special = np.array([0.0, -0.0, 65504.0, 65519.99, 65520.0, 1e9, -1e9, np.inf, -np.inf, 2.0 ** -24, 2.0 ** -25,
                        2.0 ** -25 * 1.0000001, 3 * 2.0 ** -26, 2.0 ** -14, 2.0 ** -14 * (1 - 2.0 ** -11),
                        6.1e-5, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11], np.float32)
    for x in (one_two, sweep, special, -one_two):
        code, proxy = orc.fp16_bits(x)
        with np.errstate(over="ignore"):
            ref = x.astype(np.float16)
        assert np.array_equal(code.astype(np.uint16), ref.view(np.uint16))
        assert np.array_equal(proxy, ref.astype(np.float32))
    nan_code, _ = orc.fp16_bits(np.array([np.nan], np.float32))
    assert (nan_code[0] & 0x7C00) == 0x7C00 and (nan_code[0] & 0x3FF) != 0
