# PDL trigger placement A/B at n=2, eager bf16 2-64 MiB: plain / PDL early trigger / PDL late trigger
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
MID=$(python -c "print(','.join(str(1024<<k) for k in (11,12,13,14,16)))")
i=0
for env in "HFR_PDL=0" "HFR_PDL=2" "HFR_PDL=2 HFR_PDL_LATE=1" "HFR_PDL=0" "HFR_PDL=2 HFR_PDL_LATE=1"; do
  i=$((i+1))
  env $env timeout 200 $R --master-port $((29830+i)) tools/sweep.py --dtype bf16 --sizes $MID --algos auto 2>/dev/null | grep '^{' | sed "s/^{/{\"env\": \"$env\", /" >> gpurun_out/l_pdl.jsonl; echo "$env rc=$?"
done
python - <<'PY'
import json, collections
t = collections.defaultdict(list)
for l in open("gpurun_out/l_pdl.jsonl"):
    d = json.loads(l); t[d["env"]].append((d["bytes"] >> 20, round(d["us"], 2)))
for k, v in t.items(): print(k, v)
PY
