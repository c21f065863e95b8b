"""Summarise an .ncu-rep: key metrics per kernel, opcode mix, stall reasons and the hottest
source lines (diagnostic).  usage: python tools/ncu_summary.py REPORT [kernel-substring] [nlines]"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy", "Issued Instructions",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Achieved Active Warps Per SM",
        "Registers Per Thread", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size"]


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return 0.0


def main(rep, kname="", nlines=30):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    seen = collections.OrderedDict()
    for x in rows[1:]:
        d = dict(zip(h, x))
        if kname not in d["Kernel Name"]:
            continue
        key = (d["ID"], d["Kernel Name"][:60])
        if d["Metric Name"] in KEYS:
            seen.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
    for key, m in seen.items():
        print(key)
        for k in KEYS:
            if k in m:
                print("   %-40s %s" % (k, m[k]))
    ids = [k[0] for k in seen]
    for kid in ids[:4]:
        txt = ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", "0",
                  "--print-kernel-base", "function", "--kernel-id", f"::regex:.*:{int(kid) + 1}")
        r = list(csv.reader(io.StringIO(txt)))
        hdr = next((x for x in r if x and x[0] == "Line No"), None)
        if not hdr:
            continue
        ie, iw = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        line, samp, src = collections.Counter(), collections.Counter(), {}
        cur, f = None, ""
        for x in r:
            if x and x[0] == "File Path":
                f = x[1].split("/")[-1]
                continue
            if not x or not (x[0].isdigit() or x[0] in ("-", "")):
                continue
            if x[0].isdigit():
                cur = (f, int(x[0]))
                src[cur] = x[1]
            if len(x) > ie:
                line[cur] += num(x[ie])
                samp[cur] += num(x[iw])
        tot, ts = sum(line.values()) or 1, sum(samp.values()) or 1
        print("kernel id", kid, "instructions", int(tot))
        for k, v in sorted(samp.items(), key=lambda a: -a[1])[:int(nlines)]:
            print("  %-18s %5.1f%% samples %5.1f%% inst  %s" % (f"{k[0][:10]}:{k[1]}", 100 * v / ts, 100 * line[k] / tot,
                                                                src.get(k, "")[:80]))


if __name__ == "__main__":
    main(*sys.argv[1:])
