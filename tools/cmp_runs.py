"""Print the key numbers of bench.py JSON lines and their Gantt dumps.

    python tools/cmp_runs.py gpurun_out/a.json[:spans.json] ...
"""
import json
import subprocess
import sys
from collections import defaultdict

for arg in sys.argv[1:]:
    path, _, spans = arg.partition(":")
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "ERR", e)
        continue
    pk = d.get("per_kernel_ms", {})
    print(f"{path}: {d['value']:.1f} tok/s  {d['ms_per_step']:.2f} ms  hit {d.get('hit_ratio', 0):.3f}  "
          f"gather frac {d['roofline']['frac']:.3f}  in-step {d['pcie_in_step_frac']['of_memcpy_peak']:.3f}  "
          + " ".join(f"{k}={v:.2f}" for k, v in sorted(pk.items())))
    if spans:
        sp = json.load(open(spans))
        acc = defaultdict(list)
        for n, l, a, b in sp:
            if l >= 2:
                acc[n].append((b - a) * 1000)
        print("   concurrent us/layer: " + " ".join(f"{n}:{sum(v) / len(v):.0f}" for n, v in sorted(acc.items())))
        print("   " + subprocess.run([sys.executable, "tools/spans.py", spans], capture_output=True,
                                     text=True).stdout.strip().splitlines()[-1])
