"""Reading the oracle-only golden records of tests/golden/<cfg>_gmres.json (written by scripts/make_golden.py from
oracle/ alone) and comparing a solution with them through their seeded sketch."""
import json
import os

import numpy as np

from paper_2602_00735_b200.workloads import probe_vector

HERE = os.path.dirname(os.path.abspath(__file__))


def golden_path(name: str) -> str:
    return os.path.join(HERE, "golden", f"{name}_gmres.json")


def load_golden(name: str) -> dict:
    with open(golden_path(name)) as f:
        return json.load(f)


def as_complex(pairs) -> np.ndarray:
    a = np.asarray(pairs, np.float64)
    return a[:, 0] + 1j * a[:, 1]


def sketch(x: np.ndarray, seed: int, rows: int) -> np.ndarray:
    """s_i = sum_g S_ig x_g, S_i = probe_vector(n, seed + i) (unconjugated), as scripts/make_golden.py writes it."""
    return np.array([np.dot(probe_vector(x.size, seed + i), x) for i in range(rows)])


def sketch_rel(x: np.ndarray, g: dict, key: str = "sketch_x") -> float:
    """||S (x - x_golden)|| / ||S x_golden||."""
    ref = as_complex(g[key])
    s = sketch(np.ascontiguousarray(x, np.complex128), g["sketch_seed"], g["sketch_rows"])
    return float(np.linalg.norm(s - ref) / np.linalg.norm(ref))
