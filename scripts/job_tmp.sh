cd $GRAFT_REPO_ROOT
for S in 3 4 5 6 8 10; do echo "splits=$S $(CKV_ATTN_SPLITS=$S timeout 300 python bench.py --quick --no-cpu --steps 20 2>&1 | tail -1 | cut -c1-60)"; done
