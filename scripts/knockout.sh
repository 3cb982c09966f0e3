# Timing experiments (results invalid for knockouts): warm graph step variants.
echo "base $(timeout 300 python bench.py --quick --no-cpu --steps 10 2>&1 | tail -1 | cut -c1-60)"
echo "side_sync=0 $(CKV_SIDE_SYNC=0 timeout 300 python bench.py --quick --no-cpu --steps 10 2>&1 | tail -1 | cut -c1-60)"
for K in "$@"; do
  echo "knockout=[$K] $(CKV_KNOCKOUT=$K timeout 300 python bench.py --quick --no-cpu --steps 10 2>&1 | tail -1 | cut -c1-60)"
done
