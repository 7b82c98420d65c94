"""Single-core timings of the REFERENCE's own mmpf_pls / pls_recursive (oracle/_ref, the
reference sources compiled as shipped) on the five BASELINE configurations, on this host.

Inputs are made on the GPU by the engine (randomize / X*Y / the fixed-weight generator),
downloaded, and checked against the reference generator's digests (tests/golden/configs.json)
before the reference factors them; the reference's outputs are checked against the golden
digests too.  One thread pinned to one core (the library is single-threaded), one run per
config and path, only the mmpf_pls / pls_recursive call timed.

    python tools/ref_configs.py [names...] > profiles/r2_reference_configs_cpu.json
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1006_1744_b200 as f2  # noqa: E402
from oracle_lib import Oracle, RefLib, digest  # noqa: E402


def gpu_input(cfg, o):
    if cfg["kind"] == "dense":
        a = f2.DeviceMatrix(cfg["m"], cfg["n"])
        a.randomize(0.5, cfg["seed"])
    elif cfg["kind"] == "xy":
        x = f2.DeviceMatrix(cfg["m"], cfg["inner"])
        x.randomize(0.5, cfg["seed_x"])
        y = f2.DeviceMatrix(cfg["inner"], cfg["n"])
        y.randomize(0.5, cfg["seed_y"])
        a = f2.mul_m4rm(x, y)
    else:
        return o.fixed_weight(cfg["m"], cfg["n"], cfg["weight"], cfg["seed"])
    return a.download()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))
    names = sys.argv[1:] or ["c1_dense_4096", "c2_dense_16384", "c5_sparse_16384x131072", "c4_xy_32768",
                             "c3_dense_65536"]
    os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    o, R = Oracle(), RefLib()
    out = {"host_cpu": cpu_model(), "host_cores": os.cpu_count(), "threads": 1,
           "note": "reference mmpf_pls / pls_recursive, one thread pinned to one core, one run each; "
                   "cutoff_bytes 2 MiB; outputs checked against tests/golden/configs.json", "configs": {}}
    for name in names:
        g = gold[name]
        a = gpu_input(g, o)
        assert digest(a) == int(g["input_digest"]), name
        rec = {}
        for path in g["paths"]:
            t0 = time.perf_counter()
            if path == "mmpf":
                w, P, Q, r = R.mmpf_pls(a, g["n"])
            else:
                w, P, Q, r = R.pls_recursive(a, g["n"], int(g["cutoff_bytes"]))
            dt = time.perf_counter() - t0
            ref = g[path]
            ok = (r == ref["rank"] and digest(w) == int(ref["packed_digest"]) and digest(P) == int(ref["p_digest"])
                  and digest(Q) == int(ref["q_digest"]))
            rec[path] = {"seconds": round(dt, 3), "rank": r, "matches_golden": bool(ok)}
            print(name, path, rec[path], file=sys.stderr, flush=True)
            del w, P, Q
        out["configs"][name] = rec
        del a
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
