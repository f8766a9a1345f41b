#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one kernel of an ncu report, by joining
ncu's SASS source page with nvdisasm -g line info of the same cubin (run here, on the CPU box).

    python tools/ncu_lines.py <prof.ncu-rep> <libfoe.so> <mangled kernel name> [top]
    OUTER=1 python tools/ncu_lines.py ...   attribute inlined code to the kernel-level call-site line
"""
import collections, csv, io, os, re, subprocess, sys, tempfile


def main():
    rep, so, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    ai, ie, ss = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ai], 16), float(r[ie] or 0), float(r[ss] or 0)) for r in rows[2:] if len(r) > ss]
    base = data[0][0]
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        flag = "-gi" if os.environ.get("OUTER") else "-g"   # OUTER=1: the kernel-level (outermost) call-site line
        dis = subprocess.run(["nvdisasm", flag, os.path.join(d, cub)], capture_output=True, text=True).stdout
    sec = dis[dis.index(".text." + fn + ":"):]
    sec = sec[: sec.find("\n.text.", 10) if "\n.text." in sec[10:] else len(sec)]
    line_of = {}
    cur = None
    for L in sec.split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', L)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", L)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for a, i, s in data:
        k = line_of.get(a - base, ("?", 0))
        agg[k][0] += i
        agg[k][1] += s
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {ti:.4g}, stall samples {ts:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k[0]}:{k[1]:<5d} inst {100 * v[0] / ti:5.1f}%  samples {100 * v[1] / ts:5.1f}%")


if __name__ == "__main__":
    main()
