"""Ad-hoc timing of the engine on the dense configs (development aid)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1006_1744_b200 as f2

f2.load_library()
sizes = [int(x) for x in sys.argv[1:]] or [4096, 16384, 65536]
for n in sizes:
    a0 = f2.DeviceMatrix(n, n)
    a0.randomize(0.5, 3)
    for entry in ("recursive", "mmpf"):
        if entry == "mmpf" and n > 16384:
            continue
        for rep in range(3):
            a = a0.clone()
            f2.stats_reset()
            f2.stats_enable(rep == 2)
            t0 = time.perf_counter()
            r = f2.pls_recursive(a, f2.EliminationConfig(cutoff_bytes=2 << 20)) if entry == "recursive" else f2.mmpf_pls(a)
            dt = time.perf_counter() - t0
            f2.stats_enable(False)
            gb = 2 * n ** 3 / 3 / dt / 1e9
            line = f"n={n} {entry} rep={rep} rank={r.rank} {dt*1e3:.2f} ms  {gb:.0f} Gbit-op/s launches={f2.last_launch_count()}"
            if rep == 2:
                for k, nm in enumerate(["schur", "leafpivot", "trsm", "other"]):
                    s = f2.stats_get(k)
                    line += f"\n   {nm}: n={s['launches']} ms={s['ms']:.2f}"
                    if k == 0 and s['ms'] > 0:
                        line += f" Tbitop/s={s['bitops']/s['ms']/1e9:.1f} GB/s={s['bytes']/s['ms']/1e6:.0f}"
            print(line, flush=True)
