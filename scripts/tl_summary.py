"""Summarise a CKV_TIMELINE dump (stderr of scripts/timeline.py): per kernel name, the mean gap
from the previous kernel end to this kernel's end (us), on the main vs side streams."""
import collections, re, sys
lines = open(sys.argv[1]).read().splitlines()
rows, cur = [], None
for ln in lines:
    m = re.match(r"\[tl\]\s+([\d.]+) us\s+\+\s*([\d.-]+)\s+(\S+)", ln)
    if m:
        cur = [float(m.group(1)), float(m.group(2)), m.group(3), None]
        rows.append(cur)
    m2 = re.match(r"\[tl-stream\] (\S+)", ln)
    if m2 and cur is not None:
        cur[3] = m2.group(1)
streams = collections.Counter(r[3] for r in rows)
main = streams.most_common(1)[0][0]
d = collections.defaultdict(list)
last = {}
for t, _, name, st in rows:
    prev = last.get(st)
    if prev is not None:
        d[(st == main, name)].append(t - prev)
    last[st] = t
span = rows[-1][0] - rows[0][0]
print(f"span {span:.1f} us over {len(rows)} launches")
for (is_main, name), v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{'main' if is_main else 'side'} {name:40s} n={len(v):4d} mean_gap={sum(v)/len(v):7.2f} total={sum(v):8.1f}")
