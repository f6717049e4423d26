"""Golden output-format fixtures, made by the REFERENCE:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_harness.py

Feeds fixed IterationRecord / RunSummary values (including None fields and
floats that need repr round-tripping) through antbatch.bench.write_records_csv
and summary_json_text and stores the exact text (cpu_count masked).
"""

import json
import os
import sys
from types import SimpleNamespace

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from antbatch.bench import (ExperimentConfig, IterationRecord, RunSummary, SyntheticSpec,  # noqa: E402
                            records_csv_text, summary_json_text)
from antbatch.model import AcoParams, GammaSchedule, Selection  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

RECORDS = [
    (0, 5, 0, 1.25, 1234.5, 1234.5, 3.1, 1.5, 0.1),
    (0, 5, 1, 0.1 + 0.2, 1200.0, 1200.0, None, 1.4268, 0.1),
    (1, 6, 0, 2.0, 987.654321, 987.654321, None, None, 0.25),
]
SUMMARIES = [
    (0, 5, 2, 1200.0, 0.5, 1, 0.30000000000000004, "max_iters"),
    (1, 6, 1, 987.654321, None, 0, 2.0, "time_limit"),
]


def main():
    config = ExperimentConfig(
        params=AcoParams(m=8, k=2, alpha=1.0, beta=2.0, rho=0.1, selection=Selection.ADAIR,
                         gamma_schedule=GammaSchedule(1.5, 1.0, 7), max_iters=2, seed=5),
        synthetic=SyntheticSpec(n=12, seed=1, kind="uniform"), repetitions=2, best_known=1000.0)
    inst = SimpleNamespace(name="rnd12", n=12, best_known=1000.0)
    recs = [IterationRecord(*r) for r in RECORDS]
    sums = [RunSummary(*r) for r in SUMMARIES]
    with open(os.path.join(HERE, "harness_records.csv"), "w") as f:
        f.write(records_csv_text(recs))
    doc = json.loads(summary_json_text(config, inst, sums))
    doc["aggregate"]["cpu_count"] = None
    with open(os.path.join(HERE, "harness_summary.json"), "w") as f:
        f.write(json.dumps(doc, indent=2, sort_keys=True) + "\n")
    print("wrote harness_records.csv, harness_summary.json")


if __name__ == "__main__":
    main()
