"""Writes tests/golden/oracle_digests.json: SHA-256 digests of the ORACLE's outputs on seeded small
inputs ("golden buffer recorded once ... and checked thereafter").  Calls only
oracle/ and pmg_inputs (never the CUDA path).  Re-run only when a change to the oracle's arithmetic is
justified by a PAPER.md passage or DESIGN.md reading (name it in the commit message).

    python tests/golden/make_golden.py
"""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import pmg_inputs as PI  # noqa: E402
from oracle import evaluate  # noqa: E402

CASES = [("blur", 32, 32), ("harris", 32, 32), ("unsharp", 32, 32), ("camera", 64, 48),
         ("local_laplacian", 256, 128)]


def digests():
    out = {}
    for name, W, H in CASES:
        w = PI.small(name, W, H)
        for variant in ("uniform", "structured"):
            res = evaluate(w.text, w.params, w.inputs(variant))
            for k, v in res.items():
                out[f"{name}/{W}x{H}/{variant}/{k}"] = hashlib.sha256(v.tobytes()).hexdigest()
    return out


if __name__ == "__main__":
    path = Path(__file__).with_name("oracle_digests.json")
    path.write_text(json.dumps(digests(), indent=1, sort_keys=True) + "\n")
    print(path)
