R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
SZ=$(python -c "print(','.join(str(1024<<k) for k in range(5,11)))")
for dt in bf16 f32; do
HFR_LL_MAX=$((8<<20)) timeout 900 $R --nproc-per-node 4 --master-port 31411 tools/sweep.py --graph --iters 50 --dtype $dt --oneshot-max $((8<<20)) --sizes $SZ --algos oneshot,flat --out gpurun_out/ll2_$dt.jsonl > /dev/null 2>gpurun_out/ll2.err; echo sw=$?
HFR_LL_MAX=$((8<<20)) timeout 900 $R --nproc-per-node 2 --master-port 31412 tools/sweep.py --graph --iters 50 --dtype $dt --oneshot-max $((8<<20)) --sizes $SZ --algos oneshot,flat --out gpurun_out/ll2_${dt}_n2.jsonl > /dev/null 2>>gpurun_out/ll2.err
python -c "
import json
for f in ('gpurun_out/ll2_$dt.jsonl','gpurun_out/ll2_${dt}_n2.jsonl'):
    by={}
    for l in open(f):
        d=json.loads(l); by.setdefault(d['bytes'],{})[d['algo']]=round(d['us'],1); n=d['n']
    for b in sorted(by): print('$dt', n, b, by[b])"
done
