"""Parser for tests/golden/examples.txt (hand-derived examples, see its header)."""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from tpxgen import HIT_DTYPE

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "examples.txt")


@dataclass
class Example:
    eid: str
    what: str
    dt: int = 0
    width: int = 256
    height: int = 256
    hits: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=HIT_DTYPE))
    labels: list | None = None
    global_labels: list | None = None
    static_labels: list | None = None
    features: list = field(default_factory=list)
    nclusters: int | None = None


def load() -> list[Example]:
    out: list[Example] = []
    cur: Example | None = None
    with open(PATH) as f:
        for raw in f:
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            key, _, rest = line.partition(" ")
            if key == "example":
                eid, _, what = rest.partition(" ")
                cur = Example(eid=eid, what=what)
                out.append(cur)
            elif key == "sensor":
                w, h = rest.split()
                cur.width, cur.height = int(w), int(h)
            elif key == "dt":
                cur.dt = int(rest)
            elif key == "hits":
                rows = [tuple(int(v) for v in tok.split(",")) for tok in rest.split()]
                h = np.zeros(len(rows), dtype=HIT_DTYPE)
                for i, r in enumerate(rows):
                    h[i]["x"], h[i]["y"], h[i]["toa"] = r[0], r[1], r[2]
                    h[i]["tot"] = r[3] if len(r) > 3 else 1
                cur.hits = h
            elif key == "labels":
                cur.labels = [int(v) for v in rest.split()]
            elif key == "global":
                cur.global_labels = [int(v) for v in rest.split()]
            elif key == "static":
                cur.static_labels = [int(v) for v in rest.split()]
            elif key == "feature":
                cur.features.append({k: int(v) for k, v in (t.split("=") for t in rest.split())})
            elif key == "nclusters":
                cur.nclusters = int(rest)
            else:
                raise ValueError(f"bad golden line: {line}")
    return out
