R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "dbt 65536 64" "dbt 32768 148" "pair_dbt 65536 64"; do
set -- $cfg
i=$((i+1))
timeout 600 $R --nproc-per-node 4 --master-port $((29900+i)) tools/tree_trace.py --algo $1 --chunk $2 --ctas $3 --out gpurun_out/tr_$1_$2_$3 2>gpurun_out/tr_$i.err | grep '^{'
python tools/tree_trace.py --analyze gpurun_out/tr_$1_$2_$3 > gpurun_out/tr_$1_$2_$3/summary.json
done
