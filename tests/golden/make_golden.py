"""Generate tests/golden/golden.json from the CPU oracle (portable normals).

The reference ships no stored outputs, so these fixtures pin
the oracle's results for fixed seeds; tests/test_golden.py checks the oracle
(CPU) and the GPU library (on the B200) against them.  Re-run after an
intentional change of the oracle:  python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def text(name):
    for d in (os.path.join(HERE, "scenarios"), os.path.join(ROOT, "scenarios")):
        p = os.path.join(d, name + ".json")
        if os.path.exists(p):
            return open(p).read()
    raise FileNotFoundError(name)


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def variant(name, **kw):
    j = json.loads(text(name))
    j.update(kw)
    return json.dumps(j)


def main():
    oracle.build()
    out = {}
    oracle.set_normal_mode(oracle.PORTABLE)
    keys = np.arange(256, dtype=np.uint64)
    out["normals_seed1_portable_bits"] = [int(x) for x in oracle.normals(1, keys, 0, 0).view(np.uint64)]
    oracle.set_normal_mode(oracle.GLIBC)
    out["normals_seed1_glibc_bits"] = [int(x) for x in oracle.normals(1, keys, 0, 0).view(np.uint64)]
    oracle.set_normal_mode(oracle.PORTABLE)

    banks = {}
    for name, T, n in (("minimal", 32, 64), ("quad3d_three_obstacle", 64, 32)):
        cl, _ = oracle.scenario_models(text(name))
        b = oracle.presample_bank(cl, T, n, 1, workers=4)
        banks[name] = {"T": T, "n": n, "seed": 1, "sha256": digest(b), "first": float(b[1, 0, 0]),
                       "last_bits": int(b[-1, -1, -1:].view(np.uint64)[0])}
    out["banks"] = banks

    runs = {}
    for name, kw in (("minimal", {"mc_samples": 4000}), ("three_obstacle", {"mc_samples": 4000}),
                     ("quad3d_three_obstacle", {"samples": 600, "mc_samples": 4000})):
        t = variant(name, **kw)
        r = oracle.run_pump(t, workers=os.cpu_count() or 4)
        runs[name] = {"overrides": kw, "success": int(r["success"]), "path": r["path"].tolist(),
                      "cost_bits": int(np.float64(r["cost"]).view(np.uint64)),
                      "certified_cp": r["certified_cp"], "cp_hat": r["cp_hat"],
                      "partial_plans": int(r["partial_plans"]), "termination": r["termination"],
                      "mc_eval_ids": r["mc_eval_ids"].tolist(), "mc_eval_values": r["mc_eval_values"].tolist(),
                      "pareto_cp": r["pareto_cp"].tolist(), "smoothing_s": r["smoothing_s"],
                      "traj_sha256": digest(r["traj_t"], r["traj_pos"], r["traj_vel"], r["traj_ctrl"])}
    out["runs"] = runs
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote golden.json")


if __name__ == "__main__":
    main()
