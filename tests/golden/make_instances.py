"""Golden instance-builder vectors, made by running the
REFERENCE itself in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_instances.py

Records, from antbatch's own builders:
  * the synthetic specs' coordinates and dist/eta (bench.make_synthetic_instance
    + bench.load_instance, bench.py:127-159: numpy draws, 1-decimal rounding,
    EUC_2D through model.build_instance);
  * dist/eta of one coordinate set under each TSPLIB convention (EUC_2D,
    CEIL_2D, ATT: tsplib.distance tsplib.py:198-215) and the unrounded
    euclidean_instance (model.py:124-134);
  * a degenerate set (a duplicate point and a pair < 0.5 apart, zero only
    after EUC_2D rounding): the DegenerateInstance message and the lenient eta.
Output: tests/golden/reference_instances.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import antbatch  # noqa: E402
from antbatch.bench import ExperimentConfig, SyntheticSpec, load_instance, make_synthetic_instance  # noqa: E402
from antbatch.model import AcoParams, DegenerateInstance  # noqa: E402
from antbatch.tsplib import RawTspFile  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

SPECS = [("clustered", 53, 3), ("uniform", 41, 1)]


def raw_of(coords: np.ndarray, kind: str) -> RawTspFile:
    return RawTspFile(name="", dimension=len(coords), edge_weight_type=kind,
                      node_coords=tuple((i + 1, float(x), float(y)) for i, (x, y) in enumerate(coords)))


def main() -> None:
    out = {}
    params = AcoParams(m=4, k=1)
    for kind, n, seed in SPECS:
        spec = SyntheticSpec(n=n, seed=seed, kind=kind)
        raw = make_synthetic_instance(spec)
        inst = load_instance(ExperimentConfig(params=params, synthetic=spec))
        tag = f"syn_{kind}{n}"
        out[f"{tag}/spec"] = np.array([n, seed])
        out[f"{tag}/coords"] = np.array([(x, y) for _, x, y in raw.node_coords])
        out[f"{tag}/dist"] = inst.dist
        out[f"{tag}/eta"] = inst.eta

    # one coordinate set (continuous, so ATT / CEIL_2D / EUC_2D all differ)
    g = np.random.default_rng(77)
    coords = g.uniform(0.0, 3000.0, size=(37, 2))
    out["conv/coords"] = coords
    for kind in ("EUC_2D", "CEIL_2D", "ATT"):
        inst = antbatch.build_instance(raw_of(coords, kind))
        out[f"conv/{kind}/dist"] = inst.dist
        out[f"conv/{kind}/eta"] = inst.eta
    inst = antbatch.euclidean_instance(coords)
    out["conv/EXACT/dist"] = inst.dist
    out["conv/EXACT/eta"] = inst.eta

    # degenerate: cities 2 and 9 coincide; 1 and 3 are 0.3 apart (EUC_2D -> 0)
    d = g.uniform(0.0, 500.0, size=(12, 2))
    d[9] = d[2]
    d[3] = d[1] + np.array([0.3, 0.0])
    out["degen/coords"] = d
    for kind in ("EUC_2D", "EXACT"):
        try:
            if kind == "EXACT":
                antbatch.euclidean_instance(d)
            else:
                antbatch.build_instance(raw_of(d, kind))
            msg = ""
        except DegenerateInstance as e:
            msg = str(e)
        out[f"degen/{kind}/message"] = np.array(msg)
        inst = (antbatch.euclidean_instance(d, lenient=True) if kind == "EXACT"
                else antbatch.build_instance(raw_of(d, kind), lenient=True))
        out[f"degen/{kind}/dist"] = inst.dist
        out[f"degen/{kind}/eta"] = inst.eta
    path = os.path.join(HERE, "reference_instances.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
