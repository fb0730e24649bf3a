"""Measure B200 cost tables for the scheduler (see gpu/calibrate.py) and
write them as JSON: python tools/calibrate.py [--model llama3-8b] [--out F]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2512_14142_b200.gpu.calibrate import calibrate  # noqa: E402
from paper_2512_14142_b200.gpu.datapath import KvDataPath  # noqa: E402
from paper_2512_14142_b200.gpu.model import PRESETS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--out", default="gpurun_out/b200_cost_tables.json")
a = ap.parse_args()
dp = KvDataPath(PRESETS[a.model], num_blocks=16 * 34 + 160)
cal = calibrate(dp)
Path(a.out).parent.mkdir(parents=True, exist_ok=True)
Path(a.out).write_text(json.dumps(cal, indent=1))
print(json.dumps(cal))
