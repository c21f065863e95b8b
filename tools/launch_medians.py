"""Per-kernel median launch time (us) of an ncu --metrics gpu__time_duration.sum launch list of
bench.py, restricted to the pegase launches (before the time-to-residual case9 context, i.e. the
fourth k_init).  usage: python tools/launch_medians.py launches.csv"""
import collections
import csv
import statistics
import sys


def medians(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    seq = []
    for r in rows[hdr + 1:]:
        try:
            seq.append((int(r[ii]), r[ki].split("(")[0].replace("void ", "").split("::")[-1], float(r[vi].replace(",", ""))))
        except (ValueError, IndexError):
            continue
    seq.sort()
    d, inits = collections.defaultdict(list), 0
    for _, name, v in seq:
        if name == "k_init":
            inits += 1
            if inits == 4:
                break
        if name.startswith("k_") and name != "k_init":
            d[name].append(v / 1e3)
    return {k: (statistics.median(v), len(v)) for k, v in d.items()}


if __name__ == "__main__":
    for k, (m, n) in sorted(medians(sys.argv[1]).items(), key=lambda kv: -kv[1][0]):
        print(f"| {k} | {m:.1f} | {n} |")
