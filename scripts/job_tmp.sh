cd $GRAFT_REPO_ROOT
for SS in 1 0; do
CKV_SIDE_SYNC=$SS timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_ss$SS.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ss$SS.log').read().strip().splitlines()[-1]); c=d['cold_cache']; print('side_sync=$SS', round(d['us_per_layer'],1), 'cold', round(c['us_per_layer'],1), 'link', round(c['link_gbs'],1), 'exposed', round(c['exposed_gather_us_per_layer'],1), 'period', round(d['paper_period']['us_per_layer'],1), 'e2e', round(d['e2e']['value'],1))"
done
