cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{
echo "noprefetch $(timeout 300 python bench.py --quick --no-cpu --steps 10 --no-prefetch 2>&1 | tail -1 | cut -c1-80)"
bash scripts/knockout.sh score_tc row_lse chunk_sum topk_scores cache_plan gather compact_kv attn_tc attn_combine epoch_inc
} > gpurun_out/knockout.log 2>&1
cat gpurun_out/knockout.log
