R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in "4096 2" "8192 1" "8192 2" "2048 2" "2048 4" "4096 3"; do
set -- $cfg
HFR_TMA_TILE=$1 HFR_TMA_PER_SM=$2 timeout 300 python tools/sweep.py --virtual 8 --sizes $((186<<20)) --algos flat > gpurun_out/tt.json 2>/dev/null; python -c "
import json; x=json.loads(open('gpurun_out/tt.json').read().strip().splitlines()[-1]); print('v8 $cfg', round(x['busbw'],1))"
HFR_TMA_TILE=$1 HFR_TMA_PER_SM=$2 timeout 300 $R --nproc-per-node 4 --master-port $((30600+$1/1024+$2)) tools/sweep.py --dtype bf16 --sizes $((1<<30)) --algos flat > gpurun_out/tt.json 2>/dev/null; python -c "
import json; x=json.loads(open('gpurun_out/tt.json').read().strip().splitlines()[-1]); print('n4 $cfg', round(x['busbw'],1))"
done
