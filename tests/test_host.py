"""Host-side logic of the product path (no GPU): seed derivation, PCG64 jump
constants, path configuration, shape tables, argument validation."""

import numpy as np
import pytest

from oracle import rng as orng
from oracle import shapes as oshapes
from paper_2402_05396_b200 import seeds
from paper_2402_05396_b200.pipeline import PathConfig, train_range
from paper_2402_05396_b200.shapes import SHAPES, zipf_tables


def test_derive_seed_matches_reference_restatement():
    for keys in [(0, 4, 0, 1), (7, 5, 123, 2), (2**31 + 5, 4, 99)]:
        assert seeds.derive_seed(*keys) == orng.derive_seed(*keys)


def test_lcg_jump_reproduces_numpy_stream():
    rng = np.random.default_rng(4242)
    state, inc = seeds.pcg_state(rng)
    vals = rng.random(64)
    B = 9
    jm, ja = seeds.lcg_jump(B, inc)
    # position b + 1, then + B per round: the device sampler's walk
    for b in (0, 3, 8):
        m1, a1 = seeds.lcg_jump(b + 1, inc)
        s = (m1 * state + a1) & orng.M128
        for k in range(6):
            if k:
                s = (jm * s + ja) & orng.M128
            assert (orng.pcg_output(s) >> 11) * 2.0**-53 == vals[k * B + b]


def test_pcg_state_rejects_other_generators():
    with pytest.raises(ValueError):
        seeds.pcg_state(np.random.Generator(np.random.MT19937(1)))


def test_path_config_defaults_follow_runconfig():
    c = PathConfig(aggregator="tgat")
    assert (c.decoder, c.finder_policy, c.layers, c.budget) == ("gatv2", "uniform", 2, 25)
    c = PathConfig(aggregator="graphmixer", adaptive_neighbor=False)
    assert (c.decoder, c.finder_policy, c.layers, c.budget) == ("linear", "recent", 1, 10)
    with pytest.raises(ValueError):
        PathConfig(n=30, m=25)
    with pytest.raises(ValueError):
        PathConfig(finder_policy="bogus")


def test_train_range_matches_chronological_split():
    assert train_range(1000) == (0, 600)
    assert train_range(1000, window=500) == (500, 800)


def test_shape_table_matches_baseline_configs():
    assert (SHAPES["A"].V, SHAPES["A"].E, SHAPES["A"].d_e) == (9_227, 157_474, 172)
    assert (SHAPES["B"].V, SHAPES["B"].E) == (10_984, 672_447)
    assert (SHAPES["D"].V, SHAPES["D"].E) == (13_169, 1_927_145)
    assert (SHAPES["E"].V, SHAPES["E"].E, SHAPES["E"].d_e) == (16_682, 191_290_882, 186)
    assert SHAPES["C"].adaptive and SHAPES["C"].m == 25 and SHAPES["C"].n == 10 and SHAPES["C"].batch == 4000


def test_zipf_tables_host_twin_agree():
    c1, n1 = zipf_tables(500, 3)
    c2, n2 = oshapes.zipf_tables(500, 3)
    assert c1.tobytes() == c2.tobytes() and np.array_equal(n1, n2)


def test_host_shape_generator_is_sorted_and_valid():
    src, dst, ts = oshapes.synth_events(1000, 20000, 5, ts_mode=0)
    assert (np.diff(ts) >= 0).all() and ts.min() >= 0 and ts.max() < oshapes.SPAN
    assert src.min() >= 0 and src.max() < 1000 and dst.min() >= 0 and dst.max() < 1000
    # Zipf skew: the busiest source carries far more than the uniform share
    assert np.bincount(src).max() > 20 * (20000 / 1000)
    f = oshapes.synth_features(0, 10, 7, 1)
    assert f.dtype == np.float32 and f.min() >= -1.0 and f.max() < 1.0


def test_sampler_params_match_reference_store():
    """Host parameter init equals the reference ParamStore bit-for-bit
    (golden sha of every named tensor, tests/golden/scoring.npz)."""
    from test_oracle_golden import SCORING_CASES, _params_sha, scoring_inputs

    from conftest import load_golden
    from paper_2402_05396_b200.params import sampler_params
    z = load_golden("scoring")
    for tag in SCORING_CASES:
        c = scoring_inputs(z, tag)
        p = sampler_params(c["store_seed"], c["enc"], c["m"], c["d_v"], c["d_e"], c["decoder"])
        np.testing.assert_array_equal(_params_sha(p), z[f"{tag}/params_sha"], err_msg=tag)


def test_encoder_tables_match_oracle():
    from oracle import scoring as osc
    from paper_2402_05396_b200 import params
    for enc, span in ((100, 1e6), (8, 1.0), (7, 55.0)):
        a, b = params.encoder_constants(enc, span)
        assert (a, b) == osc.encoder_constants(enc, span)
        assert params.omega_table(enc, a, b).tobytes() == osc.omega(enc, a, b).tobytes()
        tab = params.freq_table(25, enc)
        assert tab.tobytes() == osc.freq_encode(np.arange(26), enc).tobytes()


def test_path_config_rejects_bad_sampler_settings():
    with pytest.raises(ValueError):
        PathConfig(precision="float16")
    with pytest.raises(ValueError):
        PathConfig(decoder="mlp")


def test_shard_bounds_cover_rows_once():
    """placement.shard_bounds: contiguous eid ranges of ceil(rows/world)
    rows that tile [0, rows) exactly; the owner of row r is r // S (the
    peer index K5 computes, rows.cuh row_source)."""
    import pytest
    from paper_2402_05396_b200.placement import shard_bounds
    for rows in (1, 7, 100, 191_290_882):
        for world in (1, 2, 3, 8):
            seen = 0
            for r in range(world):
                lo, hi, S = shard_bounds(rows, r, world)
                assert lo == min(r * S, rows) and hi - lo <= S
                seen += hi - lo
                if hi > lo:
                    assert lo // S == r and (hi - 1) // S == r
            assert seen == rows
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_fmat_host_io_matches_reference_files(tmp_path):
    """matio: files written by the reference's save_matrix (golden) load
    identically; our writer produces the same bytes; malformed files raise
    MatrixFormatError like matio.py:41-57."""
    import os
    import numpy as np
    import pytest
    from conftest import GOLDEN
    from paper_2402_05396_b200 import matio
    for name, dt in (("feat_f32.fmat", np.float32), ("feat_f64.fmat", np.float64)):
        path = os.path.join(GOLDEN, name)
        a = matio.load_matrix(path)
        assert a.dtype == dt
        out = tmp_path / name
        matio.save_matrix(out, a)
        assert out.read_bytes() == open(path, "rb").read()
        assert matio.load_features(path).dtype == np.float32
    raw = open(os.path.join(GOLDEN, "feat_f32.fmat"), "rb").read()
    for bad, msg in ((b"XMAT" + raw[4:], "bad magic"), (raw[:4] + b"\x02" + raw[5:], "unsupported version"),
                     (raw[:5] + b"\x07" + raw[6:], "element-type"), (raw[:-4], "payload size"), (raw[:10], "shorter")):
        p = tmp_path / "bad.fmat"
        p.write_bytes(bad)
        with pytest.raises(matio.MatrixFormatError, match=msg):
            matio.load_matrix(p)
    with pytest.raises(matio.MatrixFormatError):
        matio.save_matrix(tmp_path / "x.fmat", np.zeros(3, np.float32))


def test_division_free_quotient_is_correctly_rounded(tmp_path):
    """select.cu div_rn: RN(s*R) refined by one FMA residual step (R = RN(1/T))
    equals IEEE s/T -- checked on 2M random pairs incl. integer numerators."""
    import shutil
    import subprocess
    import pytest
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "mk.c"
    src.write_text(r'''
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static uint64_t s_ = 88172645463325252ull;
static uint64_t xr(void) { s_ ^= s_ << 13; s_ ^= s_ >> 7; s_ ^= s_ << 17; return s_; }
static double rnd(void) { uint64_t x = xr(); double d;
  x = (x & 0x000FFFFFFFFFFFFFull) | ((uint64_t)(1023 + (int)(xr() % 40) - 20) << 52); memcpy(&d, &x, 8); return d; }
int main(void) {
  long bad = 0;
  for (int t = 0; t < 1000; ++t) {
    double T = rnd() * (1 + (xr() % 1000000)), R = 1.0 / T;
    for (int i = 0; i < 2000; ++i) {
      double s = (i % 7 == 0) ? (double)(xr() % 5 + 1) : rnd();
      double q0 = s * R, r = fma(-q0, T, s), q1 = fma(r, R, q0);
      bad += q1 != s / T;
    }
  }
  printf("%ld\n", bad);
  return 0;
}''')
    exe = tmp_path / "mk"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(src), "-lm"], check=True)
    assert subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.strip() == "0"
