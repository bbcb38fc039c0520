#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel and grid,
splitting setup (launches before the first PCG kernel) from solve."""
import collections
import csv
import re
import sys


def main(path, out=None, setup_launches=None, align="k_max_row"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, gi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Grid Size"))
    launches = []
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void unnamed>::", "").replace("unnamed>::", "")
        launches.append((name, r[gi], float(r[vi].replace(",", ""))))
    # the window may start a few launches early (launches ncu counts and the library's counter
    # does not): align it on the setup's first kernel, then split at the library's setup count
    start = next((i for i, l in enumerate(launches) if l[0].startswith(align)), 0)
    launches = launches[start:]
    if setup_launches is not None:
        first_solve = min(int(setup_launches), len(launches))
    else:
        first_solve = next((i for i, l in enumerate(launches) if "pcg" in l[0] or "k_kstep1" in l[0]),
                           len(launches))
    lines = []
    for label, part in (("setup", launches[:first_solve]), ("solve", launches[first_solve:])):
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for name, grid, t in part:
            tot[(name, grid)] += t
            cnt[(name, grid)] += 1
        T = sum(tot.values())
        lines.append(f"== {label}: {len(part)} launches, {T / 1e6:.2f} ms kernel time")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
            lines.append(f"{v / T * 100:6.2f}% {v / 1e3:9.1f}us n={cnt[k]:4d} "
                         f"avg={v / cnt[k] / 1e3:8.1f}us {k[0][:34]:34s} {k[1]}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         sys.argv[3] if len(sys.argv) > 3 else None)
