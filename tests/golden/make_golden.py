"""Regenerate the decision-parity golden fixtures from the reference.

Run in the build container, where the reference is importable:

    python tests/golden/make_golden.py [/root/reference/pkg/src]

For every scenario in ``tests/scenarios.py`` it runs the *reference*
``agentsched.run`` and records the SHA-256 of ``RunReport.to_json()`` plus a
few human-readable fields (aggregates, event count, KV-decision counts).
Full reports for a handful of scenarios are stored gzipped so a parity
failure can be diffed field by field. The reference never travels to the
GPU box; these fixtures do.
"""

import gzip
import hashlib
import json
import sys
from collections import Counter
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")

import agentsched  # noqa: E402
import scenarios  # noqa: E402

FULL = ("c1/stateful-mlfq/12000/adaptive", "c1/stateful-mlfq/3600/adaptive",
        "c1b200/6000", "hetero/0/stateful-mlfq", "fig2/fcfs")


def summary(report):
    wl = report.audits["waste_log"]
    return {
        "sha256": hashlib.sha256(report.to_json().encode()).hexdigest(),
        "aggregates": report.aggregates(),
        "events_processed": report.audits["events_processed"],
        "kv_decisions": dict(Counter(f"{e['chosen']}:{e['reason']}" for e in wl)),
        "num_requests": len(report.per_request),
    }


def main():
    out = {}
    for name in scenarios.scenario_names():
        report = scenarios.run_scenario(agentsched, name)
        out[name] = summary(report)
        if name in FULL:
            fn = HERE / ("report_" + name.replace("/", "_") + ".json.gz")
            fn.write_bytes(gzip.compress(report.to_json().encode(), 9, mtime=0))
    meta = {"generator": "tests/golden/make_golden.py",
            "reference": "agentsched " + agentsched.__version__,
            "scenarios": out}
    (HERE / "reports.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(out)} scenarios")


if __name__ == "__main__":
    main()
