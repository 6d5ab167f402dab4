"""Pins for oracle.fp8 (E4M3 decode, NEXT-4) and the FP8 input recipe -- CPU only.

The decoder is written from the OCP E4M3 definition; it is pinned against (i) values the
format fixes by hand (largest finite 448, smallest subnormal 2^-9, smallest normal 2^-6,
1.0, the NaN codes, signed zero), (ii) a library routine -- torch's float8_e4m3fn -> float64
cast -- on all 256 codes, and (iii) monotonicity of the positive codes.  A wrong bias, a
dropped implicit bit or a subnormal exponent off by one fails (i) or (ii)."""
import numpy as np
import pytest
import torch

import oracle
import synth


def test_hand_values():
    d = oracle.e4m3_decode
    assert d([0x7E])[0] == 448.0          # S.1111.110: largest finite
    assert d([0x01])[0] == 2.0 ** -9      # smallest subnormal
    assert d([0x07])[0] == 7 * 2.0 ** -9  # largest subnormal
    assert d([0x08])[0] == 2.0 ** -6      # smallest normal
    assert d([0x38])[0] == 1.0            # e = 7 -> 2^0
    assert d([0x3C])[0] == 1.5
    assert d([0xC4])[0] == -3.0           # 1.1000.100 = -(1 + 4/8) * 2^(8-7)
    assert np.isnan(d([0x7F])[0]) and np.isnan(d([0xFF])[0])
    z = d([0x80])[0]
    assert z == 0.0 and np.signbit(z)


def test_all_codes_vs_torch():
    codes = np.arange(256, dtype=np.uint8)
    ref = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    got = oracle.e4m3_decode(codes)
    nan = np.isnan(ref)
    assert np.array_equal(nan, np.isnan(got)) and nan.sum() == 2
    assert np.array_equal(got[~nan], ref[~nan])
    assert np.array_equal(np.signbit(got[~nan]), np.signbit(ref[~nan]))


def test_positive_codes_increase():
    v = oracle.e4m3_decode(np.arange(0, 127))
    assert np.all(np.diff(v) > 0)


def test_dequantize_is_code_times_scale():
    codes = np.array([0x38, 0x3C, 0xC4, 0x00])
    assert np.array_equal(oracle.dequantize(codes, 0.25), [0.25, 0.375, -0.75, 0.0])


@pytest.mark.parametrize("dist", ["D1", "D2", "D3", "D4"])
def test_fp8_recipe(dist):
    p = synth.Problem(2, 4, 2, 128, [300, 77], dtype="fp8", dist=dist, seed=5)
    q = synth.gen_q(p)
    k = synth.fill_kv_cache(p, "k")
    v = synth.fill_kv_cache(p, "v")
    assert q.dtype == torch.bfloat16 and k.dtype == torch.float8_e4m3fn and v.dtype == torch.float8_e4m3fn
    assert p.kv_bytes == 2 * 2 * 377 * 128
    for x, s in ((k, p.k_scale), (v, p.v_scale)):
        vals = oracle.dequantize(x.view(torch.uint8).numpy(), s)
        assert np.all(np.isfinite(vals))                   # saturated, never NaN
    if dist == "D3":                                       # census codes are exact
        vals = oracle.dequantize(v.view(torch.uint8).numpy(), p.v_scale)
        assert set(np.unique(vals)) <= {0.0, float(300 // synth._census_block(p, 300)) if 300 % synth._census_block(p, 300) == 0 else 1.0,
                                        float(77 // synth._census_block(p, 77)) if 77 % synth._census_block(p, 77) == 0 else 1.0}
    elif dist == "D1":  # the cache holds the quantised values: codes x scale within E4M3's half-ulp (2^-4 rel)
        p16 = synth.Problem(2, 4, 2, 128, [300, 77], dtype="fp32", dist=dist, seed=5)
        k32 = synth.to_f64(synth.fill_kv_cache(p16, "k"))
        kq = oracle.dequantize(k.view(torch.uint8).numpy(), p.k_scale)
        live = np.abs(k32) > 2 ** -6 * p.k_scale * 2
        assert np.all(np.abs(kq - k32)[live] <= np.abs(k32)[live] * 2 ** -4 + 1e-9)
