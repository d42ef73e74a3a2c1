"""Summarise a tools/gpu_var.sh output directory: ms per step and the
permutation's phase split per library variant."""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1])
for f in sorted(d.glob("*.json")):
    ms = []
    for line in f.read_text().splitlines():
        if line.startswith("{"):
            ms.append(round(json.loads(line)["ms_per_step"], 3))
    err = d / (f.stem + ".err")
    ph = [ln for ln in err.read_text().splitlines() if "[pip" in ln] if err.exists() else []
    print(f"{f.stem:8s} {ms}  {ph[-1].split('  ')[-1] if ph else ''}")
