"""Copy the reference's three bundled 2-D scenarios into tests/golden/scenarios
(re-serialised) so parity tests can run on the GPU box, which has no
/root/reference.  Source: /root/reference/proj/scenarios/{minimal,
three_obstacle,indoor}.json.  Run from the repo root in the build container."""
import json
import os

SRC = "/root/reference/proj/scenarios"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scenarios")

if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    for name in ("minimal", "three_obstacle", "indoor"):
        with open(os.path.join(SRC, name + ".json")) as f:
            j = json.load(f)
        with open(os.path.join(DST, name + ".json"), "w") as f:
            json.dump(j, f, sort_keys=True, separators=(",", ":"))
            f.write("\n")
        print("wrote", name)
