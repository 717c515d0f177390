R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S=$((186<<20))
i=0
for L in libhfr.so libhfr_leafcopy.so; do
i=$((i+1))
export HFR_LIB=$PWD/paper_2408_14158_b200/$L
timeout 600 $R --nproc-per-node 4 --master-port $((30100+i)) tools/sweep.py --sizes $S --algos dbt,pair_dbt --chunks 32768,65536 --ctas 64,0 --out gpurun_out/t2_$L.jsonl > /dev/null 2>&1
timeout 600 $R --nproc-per-node 4 --master-port $((30110+i)) tools/tree_trace.py --algo dbt --chunk 65536 --ctas 64 --out gpurun_out/t2tr_$L 2>/dev/null | grep '^{'
python tools/tree_trace.py --analyze gpurun_out/t2tr_$L | python -c "
import json,sys
d=json.load(sys.stdin)
for r,v in sorted(d.items()):
    print('$L', r, 'span',round(v['span_us']), 'busy',round(v['cta_busy_frac_mean'],2), {k:(round(x['wait_us_sum']),round(x['work_us_mean'],1),round(x['issue_us_mean'],1),round(x['drain_us_mean'],1)) for k,x in v.items() if isinstance(x,dict)})"
done
unset HFR_LIB
for f in gpurun_out/t2_*.jsonl; do python -c "
import json
for l in open('$f'):
    d=json.loads(l); print('$f'.split('/')[-1], d['algo'], d['chunk'], d['ctas'], round(d['us'],1), round(d['busbw'],1))"; done
