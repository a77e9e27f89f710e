"""Generate the 3-D quadrotor scenarios named in BASELINE.json.

The reference ships only 2-D scenarios; these are written in its own JSON
schema (scenario.hpp:150-154) so the drop-in loader reads them unchanged.

  quad3d_three_obstacle  configs[0]: 3 boxes, n=2000, 32 particles, alpha 5%
  quad3d_indoor          configs[1]: 10 walls, n=4000, 64 particles, alpha 2%
  quad3d_forest          configs[2]: 200 boxes, n=16000, 128 particles

Run: python scenarios/make_scenarios.py  (rewrites the JSON files).
"""
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
M = (1 << 64) - 1


def mix64(x):
    x ^= x >> 30
    x = (x * 0xbf58476d1ce4e5b9) & M
    x ^= x >> 27
    x = (x * 0x94d049bb133111eb) & M
    x ^= x >> 31
    return x


def uniform(seed, a, b, c):
    """rng::uniform (rng.hpp:20-39)."""
    h = mix64((seed + 0x9e3779b97f4a7c15) & M)
    h = mix64((h + a) & M)
    h = mix64((h + b) & M)
    h = mix64((h + c) & M)
    return ((h >> 11) + 1.0) * 2.0 ** -53


def box(lo, hi):
    return {"lo": lo, "hi": hi}


def three_obstacle():
    return {
        "name": "quad3d_three_obstacle",
        "workspace": {"bounds": box([0, 0, 0], [10, 10, 4]),
                      "obstacles": [box([2.5, 0, 0], [3.5, 6.5, 4]), box([4.5, 3.5, 0], [5.5, 10, 4]),
                                    box([6.5, 0, 0], [7.5, 6.5, 4])]},
        "start": {"position": [1, 5, 2], "velocity": [0, 0, 0]},
        "goal": {"lo": [8.5, 4, 1.5], "hi": [9.5, 6, 2.5], "max_speed": 0.5},
        "noise": {"process": [0, 0, 0, 3e-4, 3e-4, 3e-4], "measurement": 5e-4, "initial": [1e-4] * 6},
        "dt": 0.2, "samples": 2000, "connection_radius": 6, "alpha": 0.05, "max_speed": 1.0,
        "particles": 32, "mc_samples": 20000, "bank_horizon": 512, "collision_resolution": 0.05,
        "seeds": {"bank": 1, "mc": 2, "rrt": 3},
    }


def indoor():
    walls2d = [([3.2, 0], [4.2, 8.0]), ([3.2, 10.0], [4.2, 12]), ([6.4, 0], [7.4, 2.0]), ([6.4, 4.0], [7.4, 12]),
               ([9.6, 0], [10.6, 8.0]), ([9.6, 10.0], [10.6, 12]), ([12.8, 0], [13.8, 2.0]),
               ([12.8, 4.0], [13.8, 12]), ([16.0, 0], [17.0, 8.0]), ([16.0, 10.0], [17.0, 12])]
    return {
        "name": "quad3d_indoor",
        "workspace": {"bounds": box([0, 0, 0], [20, 12, 3]),
                      "obstacles": [box(lo + [0], hi + [3]) for lo, hi in walls2d]},
        "start": {"position": [1.5, 6, 1.5], "velocity": [0, 0, 0]},
        "goal": {"lo": [17.5, 5, 1], "hi": [19, 7, 2], "max_speed": 0.5},
        "noise": {"process": [0, 0, 0, 2e-4, 2e-4, 2e-4], "measurement": 3e-4, "initial": [1e-4] * 6},
        "dt": 0.2, "samples": 4000, "connection_radius": 6, "alpha": 0.02, "max_speed": 1.0,
        "particles": 64, "mc_samples": 20000, "bank_horizon": 512, "collision_resolution": 0.05,
        "seeds": {"bank": 1, "mc": 2, "rrt": 3},
    }


def forest(n_boxes=200, seed=2024):
    start, goal_lo, goal_hi = [2.0, 2.0, 4.0], [36.0, 36.0, 3.0], [38.0, 38.0, 5.0]
    obstacles = []
    i = 0
    while len(obstacles) < n_boxes:
        c = [40 * uniform(seed, i, 0, 0), 40 * uniform(seed, i, 0, 1), 8 * uniform(seed, i, 0, 2)]
        e = [0.5 + 1.5 * uniform(seed, i, 0, 3 + k) for k in range(3)]
        lo = [round(c[k] - e[k] / 2, 6) for k in range(3)]
        hi = [round(c[k] + e[k] / 2, 6) for k in range(3)]
        i += 1
        # keep a 1.5 m margin around the start and the goal box
        near_start = all(lo[k] - 1.5 <= start[k] <= hi[k] + 1.5 for k in range(3))
        near_goal = all(lo[k] - 1.5 <= goal_hi[k] and goal_lo[k] <= hi[k] + 1.5 for k in range(3))
        if near_start or near_goal:
            continue
        obstacles.append(box(lo, hi))
    return {
        "name": "quad3d_forest",
        "workspace": {"bounds": box([0, 0, 0], [40, 40, 8]), "obstacles": obstacles},
        "start": {"position": start, "velocity": [0, 0, 0]},
        "goal": {"lo": goal_lo, "hi": goal_hi, "max_speed": 0.5},
        "noise": {"process": [0, 0, 0, 2e-4, 2e-4, 2e-4], "measurement": 3e-4, "initial": [1e-4] * 6},
        "dt": 0.2, "samples": 16000, "connection_radius": 4, "alpha": 0.05, "max_speed": 1.0,
        "particles": 128, "mc_samples": 20000, "bank_horizon": 1024, "collision_resolution": 0.05,
        "seeds": {"bank": 1, "mc": 2, "rrt": 3},
    }


def main():
    for sc in (three_obstacle(), indoor(), forest()):
        path = os.path.join(HERE, sc["name"] + ".json")
        with open(path, "w") as f:
            json.dump(sc, f, indent=1)
            f.write("\n")
        print("wrote", path, len(sc["workspace"]["obstacles"]), "obstacles")


if __name__ == "__main__":
    main()
