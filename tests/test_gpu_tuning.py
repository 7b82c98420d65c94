"""GPU: every alternative schedule the Tuning switches select (csrc/api.cu, struct
Tuning) stays bit-exact.  Each case runs in a fresh process (the switches are read
once, at initialisation) and checks pls_recursive, mmpf_pls and the sharded schedule
against the Gaussian oracle on dense, rank-deficient and sparse inputs."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

SCRIPT = textwrap.dedent("""
    import sys
    sys.path[:0] = [{root!r}, {here!r}]
    import numpy as np
    import paper_1006_1744_b200 as f2
    from oracle_lib import Oracle
    o = Oracle()
    cases = [(2304, 3328, o.randomize(2304, 3328, 0.5, 1)),
             (2048, 2048, o.mul(o.randomize(2048, 700, 0.5, 2), 700, o.randomize(700, 2048, 0.5, 3), 2048)),
             (1024, 8192, o.fixed_weight(1024, 8192, 4, 4))]
    for m, n, a in cases:
        w, p, q, r = o.gauss_pls(a, n)
        d = f2.DeviceMatrix.from_host(a, n)
        res = f2.pls_recursive(d, f2.EliminationConfig(cutoff_bytes=4096))
        assert res.rank == r and (res.P == p).all() and (d.download() == w).all(), ("recursive", m, n)
        assert (res.Q == o.recursive_q(m, n, 4096, q[:r])).all(), ("recursive Q", m, n)
        d = f2.DeviceMatrix.from_host(a, n)
        res = f2.mmpf_pls(d)
        assert res.rank == r and (res.P == p).all() and (res.Q == q).all() and (d.download() == w).all(), \\
            ("mmpf", m, n)
    # host buffers past the streamed-upload threshold (16 panels)
    m, n = 4096, 16384
    a = o.randomize(m, n, 0.5, 9)
    w, p, q, r = o.gauss_pls(a, n)
    h = f2.pinned_empty(a.shape)
    np.copyto(h, a)
    res = f2.pls_recursive_host(h, n, f2.EliminationConfig(cutoff_bytes=4096))
    assert res.rank == r and (res.P == p).all() and (h == w).all(), "host"
    print("ok")
""")


@pytest.mark.parametrize("env", [
    {"F2_SCHUR_M4RM": "1"},
    {"F2_NO_LOOKAHEAD": "1"},
    {"F2_NO_GRAPH": "1"},
    {"F2_NO_PDL": "1"},
    {"F2_NO_EARLY_WIDE_TRSM": "1"},
    {"F2_WIDE_EARLY_PCT": "-1", "F2_TW_JOIN": "1"},
    {"F2_WIDE_EARLY_PCT": "100"},
    {"F2_SPLIT_EARLY": "1"},
    {"F2_SPLIT_EARLY": "1", "F2_NO_EARLY_WIDE_TRSM": "1"},
    {"F2_SIDE_CTAS": "8", "F2_SIDE_CTAS_LATE": "0"},
    {"F2_LATE_PCT": "0"},
    {"F2_LATE_PCT": "100", "F2_SIDE_CTAS": "140"},
    {"F2_NO_GRAPH": "1", "F2_EVTL": "1"},
    {"F2_MMPF_PANEL_BITS": "64"},
    {"F2_MMPF_PANEL_BITS": "64", "F2_NO_LOOKAHEAD": "1"},
    {"F2_MMPF_PANEL_BITS": "256"},
    {"F2_NO_STREAM_UPLOAD": "1"},
    {"F2_UP_G0": "2", "F2_UP_PS": "14", "F2_UP_GROUPS": "11", "F2_UP_SIDE": "148"},
    {"F2_NO_GRAPH": "1", "F2_NO_EARLY_WIDE_TRSM": "1"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_tuning_switch_stays_exact(env):
    full = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, here=HERE)], env=full, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stdout[-2000:] + out.stderr[-4000:]
