"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref/libf2ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  Run here, where the
reference exists; the outputs are committed so the GPU box never needs it.

    python tests/golden/make_golden.py small     # tests/golden/small_cases.npz (seconds)
    python tests/golden/make_golden.py configs   # tests/golden/configs.json   (~10 min, 1 core)
    python tests/golden/make_golden.py io        # tests/golden/io/ (files written by io::write_*)

configs.json pins, for the five BASELINE.json configurations, the digest of the
seeded input and of the reference's packed output, P and Q, plus the rank, and
(configs up to 2^31 bits) the digest of rref_from_pls applied to the recursive result.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Oracle, RefLib, digest, words  # noqa: E402

CUTOFF = 2 << 20  # pinned cutoff_bytes (the survey container's default)

CONFIGS = {
    "c1_dense_4096": dict(m=4096, n=4096, kind="dense", seed=1, paths=["mmpf"]),
    "c2_dense_16384": dict(m=16384, n=16384, kind="dense", seed=2, paths=["recursive"]),
    "c3_dense_65536": dict(m=65536, n=65536, kind="dense", seed=3, paths=["recursive"]),
    "c4_xy_32768": dict(m=32768, n=32768, kind="xy", inner=16384, seed_x=41, seed_y=42, paths=["recursive", "mmpf"]),
    "c5_sparse_16384x131072": dict(m=16384, n=131072, kind="fixed_weight", weight=64, seed=5, paths=["recursive", "mmpf"]),
}


def make_input(cfg, o, R):
    if cfg["kind"] == "dense":
        return R.randomize(cfg["m"], cfg["n"], 0.5, cfg["seed"])
    if cfg["kind"] == "xy":
        x = R.randomize(cfg["m"], cfg["inner"], 0.5, cfg["seed_x"])
        y = R.randomize(cfg["inner"], cfg["n"], 0.5, cfg["seed_y"])
        return R.mul_m4rm(x, cfg["inner"], y, cfg["n"])
    if cfg["kind"] == "fixed_weight":
        return o.fixed_weight(cfg["m"], cfg["n"], cfg["weight"], cfg["seed"])
    raise ValueError(cfg["kind"])


def configs(only=None):
    o, R = Oracle(), RefLib()
    path = os.path.join(HERE, "configs.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name, cfg in CONFIGS.items():
        if only and name not in only:
            continue
        t0 = time.time()
        a = make_input(cfg, o, R)
        rec = dict(cfg)
        rec["cutoff_bytes"] = CUTOFF
        rec["input_digest"] = str(digest(a))
        rec["gen_s"] = round(time.time() - t0, 2)
        for p in cfg["paths"]:
            t1 = time.time()
            if p == "mmpf":
                w, P, Q, r = R.mmpf_pls(a, cfg["n"])
            else:
                w, P, Q, r = R.pls_recursive(a, cfg["n"], CUTOFF)
            dt = time.time() - t1
            rec[p] = dict(rank=int(r), packed_digest=str(digest(w)), p_digest=str(digest(P)),
                          q_digest=str(digest(Q)), q_prefix_identity=bool((Q[:r] == np.arange(r, dtype=np.uint64)).all()),
                          q_tail_nonidentity=int((Q[r:] != np.arange(r, cfg["n"], dtype=np.uint64)).sum()),
                          ref_seconds=round(dt, 2))
            if p == "recursive" and cfg["m"] * cfg["n"] <= (1 << 31):
                t2 = time.time()
                rf = R.rref_from_pls(w, cfg["n"], r, Q[:r])
                rec[p]["rref_digest"] = str(digest(rf))
                rec[p]["rref_seconds"] = round(time.time() - t2, 2)
                del rf
            print(name, p, rec[p], flush=True)
            del w, P, Q
        out[name] = rec
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)
        del a


def small():
    """Random small cases: input, and the reference's outputs for gauss / mmpf /
    recursive (several cutoffs).  Shapes and densities follow the reference's
    own randomized suites (test_mmpf.cpp:157-180, test_pls.cpp:51-79)."""
    R = RefLib()
    rng = np.random.default_rng(20261020)
    cases = []
    shapes = [(1, 1), (2, 2), (1, 200), (200, 1), (64, 64), (65, 63), (128, 130), (300, 70), (70, 300),
              (257, 257), (40, 12), (12, 40), (513, 129), (100, 1000)]
    dens = [0.02, 0.1, 0.5, 0.9]
    for i in range(60):
        if i < len(shapes):
            m, n = shapes[i]
        else:
            m, n = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        d = dens[i % 4]
        seed = int(rng.integers(1, 2 ** 62))
        a = R.randomize(m, n, d, seed)
        cut = [8, 64, 4096, 1 << 30][i % 4]
        wm, Pm, Qm, rm = R.mmpf_pls(a, n)
        wr, Pr, Qr, rr = R.pls_recursive(a, n, cut)
        rf = R.rref_from_pls(wr, n, rr, Qr[:rr])       # rref_via_pls, test_pls.cpp:21-25
        gr, grr = R.gauss_rref(a, n)                   # gauss_rref, gauss.cpp:7-23
        assert grr == rr and (gr == rf).all()
        cases.append(dict(m=m, n=n, density=d, seed=seed, cutoff=cut, a=a, mm_w=wm, mm_p=Pm, mm_q=Qm, mm_r=rm,
                          rc_w=wr, rc_p=Pr, rc_q=Qr, rc_r=rr, rref_w=rf))
    flat = {}
    for i, c in enumerate(cases):
        for k, v in c.items():
            flat[f"{i}_{k}"] = np.asarray(v)
    flat["count"] = np.asarray(len(cases))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **flat)
    print("wrote", len(cases), "small cases")


def io_fixtures():
    """Files written by the reference's io::write_matrix / write_permutation
    (io.cpp) + the words they hold: tests/golden/io/."""
    import ctypes as C
    R = RefLib()
    d = os.path.join(HERE, "io")
    os.makedirs(d, exist_ok=True)
    u64p = C.POINTER(C.c_uint64)
    R.lib.ref_write_matrix.argtypes = [C.c_char_p, u64p, C.c_size_t, C.c_size_t, C.c_int]
    R.lib.ref_write_permutation.argtypes = [C.c_char_p, u64p, C.c_size_t]
    rng = np.random.default_rng(1744)
    shapes = [(2, 3), (1, 65), (0, 5), (3, 0), (1, 1), (7, 64), (9, 130), (33, 200), (40, 127), (5, 1000)]
    flat = {}
    for i, (m, n) in enumerate(shapes):
        a = R.randomize(m, n, [0.4, 0.5, 0.1][i % 3], int(rng.integers(1, 2 ** 62)))
        if (m, n) == (2, 3):
            a = np.array([[0b101], [0b010]], np.uint64)          # test_io.cpp:12-21
        if (m, n) == (1, 65):
            a = np.array([[1, 1]], np.uint64)                     # test_io.cpp:23-39
        flat[f"m{i}"] = a
        flat[f"n{i}"] = np.asarray(n)
        for fmt, ext in [(0, "txt"), (1, "bmf2")]:
            path = os.path.join(d, f"mat{i}_{m}x{n}.{ext}").encode()
            buf = np.ascontiguousarray(a) if a.size else np.zeros(1, np.uint64)
            assert R.lib.ref_write_matrix(path, buf.ctypes.data_as(u64p), m, n, fmt) == 0
    flat["count"] = np.asarray(len(shapes))
    np.savez_compressed(os.path.join(d, "matrices.npz"), **flat)
    p = np.array([2, 1, 2, 3], np.uint64)                         # test_io.cpp:81-89
    assert R.lib.ref_write_permutation(os.path.join(d, "perm4.txt").encode(), p.ctypes.data_as(u64p), 4) == 0
    print("wrote io fixtures to", d)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    if what == "small":
        small()
    elif what == "io":
        io_fixtures()
    else:
        configs(sys.argv[2:] or None)
