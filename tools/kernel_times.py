"""A/B per-kernel timing of library variants (GPU box).

    python tools/kernel_times.py [--config c4] [--reps 10] [--rounds 5] lib1.so lib2.so ...

Each library runs in its own process (the library is bound at import via
SFEM_LIB); prints the median per-sweep-kernel times and a checksum of one
solve so that a variant that changes results is visible at a glance.
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(config, reps, rounds):
    sys.path.insert(0, HERE)
    import numpy as np
    import torch

    import bench
    import paper_1701_03967_b200 as sfem

    orders, elements, lengths, coeffs, shift, _ = bench.CONFIGS[config]
    plan = sfem.Plan(sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs))
    shape = list(plan.extents[:-1]) + [plan.pitch]
    g = torch.Generator(device="cuda").manual_seed(0)
    d = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 0.5
    d[..., plan.extents[-1]:] = 0
    x = d.clone()
    plan.solve_device(x.data_ptr())
    torch.cuda.synchronize()
    chk = float(x[..., : plan.extents[-1]].double().norm())
    per, tot = [], []
    for _ in range(rounds):
        t, k = plan.solve_device_timed(d.data_ptr(), reps)
        tot.append(t / reps if t > reps * 0.05 else t)
        per.append(k)
    per = np.median(np.array(per), axis=0)
    print(json.dumps({"kernel_ms": [round(v, 4) for v in per], "sum_ms": round(float(per.sum()), 4),
                      "checksum": chk}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.config, a.reps, a.rounds)
        return
    for lib in a.libs or [""]:
        env = dict(os.environ)
        if lib:
            env["SFEM_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, __file__, "--child", "--config", a.config, "--reps", str(a.reps),
                            "--rounds", str(a.rounds)], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr.strip()[-300:]
        print(f"{os.path.basename(lib) or 'in-tree'}: {line}", flush=True)


if __name__ == "__main__":
    main()
