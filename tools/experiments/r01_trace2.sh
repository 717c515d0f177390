R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for a in dbt pair_dbt; do
timeout 600 $R --nproc-per-node 4 --master-port 30960 tools/tree_trace.py --algo $a --chunk 32768 --ctas 0 --out gpurun_out/trc_$a 2>/dev/null | grep '^{'
python tools/tree_trace.py --analyze gpurun_out/trc_$a | python -c "
import json,sys
d=json.load(sys.stdin)
for r,v in sorted(d.items()):
    print('$a', r, 'span',round(v['span_us']), 'busy',round(v['cta_busy_frac_mean'],2), {k:(x['n'], round(x['wait_us_sum']),round(x['work_us_mean'],1),round(x['issue_us_mean'],1),round(x['drain_us_mean'],1), round(x['first_done_us']), round(x['last_done_us'])) for k,x in v.items() if isinstance(x,dict)})"
done
