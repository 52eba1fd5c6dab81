#!/usr/bin/env python
"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_shares.py LAUNCHES.csv OUT.md "command line"
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(src, errors="replace")) if len(r) >= 15 and r[0].isdigit()]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        name = r[4]
        m = re.match(r"(?:void )?([\w:]+(?:<[^(]*>)?)", name)
        k = m.group(1) if m else name
        tot[k] += float(r[14]) / 1e6
        cnt[k] += 1
    total = sum(tot.values())
    lines = [f"# Launch list shares (`ncu --metrics gpu__time_duration.sum --clock-control none`, `{cmd}`)", "",
             "Cold-cache, serialised per-launch times of every kernel the command launched (warm-up, timed, "
             "variant, attribution and e2e passes): the SHARE of each kernel is what compares with the bench "
             "line's attribution, not the absolute.", "",
             f"{len(rows)} launches, {total:.1f} ms in total.", "",
             "| kernel | launches | ms (all launches) | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        if v / total < 0.00005:
            continue
        lines.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {v / total:.3f} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
