#!/bin/bash
# Host-link gather tuning: cold whole-record loads (ra_study, aligned 16-token store and 64-token
# store) for several gather grid sizes.  Prints median link GB/s per (grid, store block).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for B in 32 64 148 296 592; do
  CKV_LIBRARY=tuning CKV_GATHER_BLOCKS=$B timeout 300 python scripts/ra_study.py --requests 3 --out gpurun_out/gs_$B.json > /dev/null 2>&1
  python - "$B" <<'PY'
import json, statistics, sys
B = sys.argv[1]
d = json.load(open(f"gpurun_out/gs_{B}.json"))
for key in [(16, 16), (1, 64)]:
    rs = [r for r in d["rows"] if (r["selection_unit"], r["store_block"]) == key]
    print(f"blocks={B:>4} sel={key[0]:>2} store={key[1]:>2} link_GBs={statistics.median(r['link_GBs'] for r in rs):6.1f} "
          f"us={statistics.median(r['gather_us'] for r in rs):7.1f}")
PY
done
