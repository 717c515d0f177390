# FLAT-TMA tile / CTAs-per-SM sweep at n=4: bf16 2-256 MiB and C2 fp32 186 MiB
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/sweep.py"
SZ=$((2<<20)),$((4<<20)),$((8<<20)),$((16<<20)),$((32<<20)),$((64<<20)),$((256<<20))
for cfg in "4096 2" "4096 1" "8192 1" "16384 1"; do
  set -- $cfg; tile=$1; psm=$2
  for dt in bf16 f32; do
    if [ $dt = bf16 ]; then S=$SZ; else S=$((186<<20)); fi
    HFR_TMA_TILE=$tile HFR_TMA_PER_SM=$psm timeout 200 $T --sizes $S --dtype $dt --algos flat --repeats 5 2>/dev/null \
      | grep '^{' | sed "s/^{/{\"tma_tile\": $tile, \"per_sm\": $psm, /" >> gpurun_out/tma_tile_n4.jsonl
    echo "tile=$tile psm=$psm $dt rc=$?"
  done
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/tma_tile_n4.jsonl")]
tab = collections.defaultdict(dict)
for r in rows:
    tab[(r["tma_tile"], r["per_sm"])][(r["dtype"], r["bytes"])] = round(r["busbw"], 1)
for k, v in sorted(tab.items()):
    print(k, [v[s] for s in sorted(v)])
PY
