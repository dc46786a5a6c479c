"""Loaders for tests/golden (outputs of the unmodified reference, see oracle/gen_golden.py)."""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

SYNTH = ["cfg1_100k_128_w4", "cfg2_60k_128_w3", "cfg3_50k_200_w4", "cfg4_40k_256_w4",
         "cfg5_20k_512_w4"]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name: str):
    return np.load(GOLDEN / f"{name}.npz")


def small_cases():
    z = load("small_cases")
    for row in z["cases"]:
        ci, dim, wd, wq, n, nq, k = (int(v) for v in row[:7])
        scale = float(row[7])
        pre = f"c{ci}_"
        yield dict(ci=ci, dim=dim, wd=wd, wq=wq, n=n, nq=nq, k=k, scale=scale,
                   **{key: z[pre + key] for key in ("docs", "queries", "planes", "qplanes", "full",
                                                    "dists", "ids", "sims", "thr", "cand")})


def synth_case(name: str):
    """Regenerate the inputs of a synthetic golden case and verify their hashes."""
    from oracle.xfbq_oracle import synthetic_unit_rows
    z = load(name)
    n, dim, wd, wq, nq, k, sd, sq = (int(v) for v in z["meta"])
    docs = synthetic_unit_rows(n, dim, sd)
    queries = synthetic_unit_rows(nq, dim, sq)
    assert sha(docs) == str(z["docs_sha"]), "synthetic docs differ from the reference generator"
    assert sha(queries) == str(z["queries_sha"])
    return dict(n=n, dim=dim, wd=wd, wq=wq, nq=nq, k=k, scale=float(z["scale"][0]), docs=docs,
                queries=queries, z=z)
