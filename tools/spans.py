"""Summarise a CLO_BENCH_SPANS Gantt dump (one timeline step of bench.py).

    python tools/spans.py gpurun_out/spans.json

Prints, per offloaded layer, when its selection chain ended, when its gather
ran and the transfer-stream gap before it, and attributes every gap either
to the selection chain (the gather could not start earlier: its fetch list
was published after the previous gather ended) or to the graph (launch /
dependency latency after the list was ready). Totals at the end.
"""
from __future__ import annotations

import json
import sys
from collections import defaultdict


def main(path: str) -> None:
    spans = json.load(open(path))
    by = defaultdict(dict)
    for name, layer, a, b in spans:
        by[layer].setdefault(name, []).append((a, b))
    gathers = sorted((v["gather_zero_copy"][0], l) for l, v in by.items() if "gather_zero_copy" in v)
    step_end = max(b for _, _, _, b in spans)
    first = min(a for _, _, a, _ in spans)
    busy = sum(b - a for (a, b), _ in gathers)
    prev_end = first
    gap_sel = gap_graph = 0.0
    print(f"{'layer':>5} {'sel_end':>8} {'g_start':>8} {'g_end':>8} {'g_ms':>6} {'gap':>6} {'cause':>6} {'attn':>6}")
    for (a, b), l in gathers:
        sel_end = max(e for n in ("reconcile", "select_offloaded", "lookup_offloaded") for _, e in by[l].get(n, []))
        gap = max(0.0, a - prev_end)
        cause = "sel" if sel_end > prev_end + 1e-3 else "graph"
        if cause == "sel":
            gap_sel += max(0.0, sel_end - prev_end)
            gap_graph += max(0.0, a - max(sel_end, prev_end))
        else:
            gap_graph += gap
        at = by[l].get("attention", [(0, 0)])[0]
        print(f"{l:>5} {sel_end:8.3f} {a:8.3f} {b:8.3f} {b - a:6.3f} {gap:6.3f} {cause:>6} {at[1] - at[0]:6.3f}")
        prev_end = b
    tail = step_end - prev_end
    span = step_end - first
    print(f"step {span:.3f} ms; transfer busy {busy:.3f} ms ({busy / span:.1%}); "
          f"gaps waiting on selection {gap_sel:.3f} ms, on graph edges {gap_graph:.3f} ms; "
          f"after the last gather {tail:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
