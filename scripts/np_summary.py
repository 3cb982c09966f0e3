"""Summarise scripts/np_sweep.sh output: average duration, clock and cycles per variant."""
import csv, glob, re, sys
for f in sorted(glob.glob("gpurun_out/np_*.csv"), key=lambda x: int(re.findall(r"np_(\d+)", x)[0])):
    rows = [r for r in csv.reader(open(f)) if len(r) > 3 and "score_tc" in "".join(r)]
    t = [float(r[-1]) for r in rows if r[-3] == "gpu__time_duration.sum"]
    c = [float(r[-1]) for r in rows if r[-3] == "sm__cycles_elapsed.avg.per_second"]
    if t and c:
        us, ghz = sum(t) / len(t) / 1e3, sum(c) / len(c) / 1e9
        print(f"{f}: {us:.1f} us  {ghz:.3f} GHz  {us * ghz * 1e3:.0f} cycles  n={len(t)}")
