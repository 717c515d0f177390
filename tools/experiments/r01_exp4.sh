R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
S=$((186<<20))
for L in libhfr.so libhfr_hints.so; do
HFR_LIB=$PWD/paper_2408_14158_b200/$L timeout 600 python tools/sweep.py --virtual 8 --sizes $S --algos flat --out gpurun_out/e4_v8_$L.jsonl > /dev/null 2>&1
HFR_LIB=$PWD/paper_2408_14158_b200/$L timeout 600 $R --nproc-per-node 4 --master-port 29961 tools/sweep.py --sizes $S --algos flat --out gpurun_out/e4_n4_$L.jsonl > /dev/null 2>&1
done
cat gpurun_out/e4_*.jsonl | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/e4_multi.log 2>&1; echo multi=$?; tail -2 gpurun_out/e4_multi.log
i=0
for cfg in "16 1 high" "16 1 low" "8 1 high" "32 1 high" "16 0 low"; do
set -- $cfg; i=$((i+1))
HFR_SIDE_PRIORITY=$3 timeout 900 $R --nproc-per-node 4 --master-port $((29970+i)) tools/ddp_overlap.py --max-ctas $1 --gate $2 2>/dev/null | grep '^{' | cut -c1-520
done
