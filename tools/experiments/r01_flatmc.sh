timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/mc_multi.log 2>&1; echo multi=$?; grep -E "passed|failed|Error" gpurun_out/mc_multi.log | tail -3
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for mc in 1 0; do
for N in 2 4; do
HFR_FLAT_MC=$mc timeout 600 $R --nproc-per-node $N --master-port $((30200+N+10*mc)) tools/sweep.py --nvls $((2<<30)) --dtype bf16 --sizes $((64<<20)),$((1<<30)) --algos flat --out gpurun_out/mc_$mc.jsonl > /dev/null 2>&1
HFR_FLAT_MC=$mc timeout 600 $R --nproc-per-node $N --master-port $((30220+N+10*mc)) tools/sweep.py --nvls $((1<<30)) --dtype f32 --sizes $((186<<20)) --algos flat --out gpurun_out/mc_$mc.jsonl > /dev/null 2>&1
done; done
for mc in 1 0; do python -c "
import json
for l in open('gpurun_out/mc_$mc.jsonl'):
    d=json.loads(l); print('mc=$mc', d['n'], d['dtype'], d['bytes'], round(d['us'],1), round(d['busbw'],1))"; done
