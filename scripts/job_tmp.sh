cd $GRAFT_REPO_ROOT
for i in 1 2; do
echo "fused=1 $(timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"
echo "fused=0 $(CKV_FUSED_SELECT=0 timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-100)"
done
