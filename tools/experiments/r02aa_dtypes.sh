# round 2: every element type (NEXT-4) through FLAT / DBT / PAIR vs NCCL at n=4 (final library)
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for dt in f32 bf16 f16 e4m3 e5m2; do
timeout 600 $R --master-port $((29960)) tools/sweep.py --dtype $dt --algos flat,dbt,pair_dbt --nccl --sizes 67108864,1073741824 --out gpurun_out/r02aa_dtypes_n4.jsonl > gpurun_out/r02aa_$dt.log 2>&1; echo $dt=$?
done
python - <<'PY'
import json
for l in open("gpurun_out/r02aa_dtypes_n4.jsonl"):
    d = json.loads(l)
    if "unsupported" in d:
        print(d["dtype"], d["bytes"], "nccl unsupported:", d["unsupported"][:80]); continue
    print(d["dtype"], d["bytes"], d["impl"], d.get("algo", ""), round(d["us"], 1), round(d["busbw"], 1))
PY
