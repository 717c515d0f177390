# mid-size (2-64 MiB bf16) FLAT-TMA tile / CTAs-per-SM sweep at n=2
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py"
SZ=$((2<<20)),$((4<<20)),$((8<<20)),$((16<<20)),$((32<<20)),$((64<<20)),$((256<<20))
for tile in 4096 2048 1024; do
  for psm in 2 1; do
    HFR_TMA_TILE=$tile HFR_TMA_PER_SM=$psm timeout 200 $T --sizes $SZ --dtype bf16 --algos flat --repeats 5 2>/dev/null \
      | grep '^{' | sed "s/^{/{\"tma_tile\": $tile, \"per_sm\": $psm, /" >> gpurun_out/tma_tile_mid_n2.jsonl
    echo "tile=$tile psm=$psm rc=$?"
  done
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/tma_tile_mid_n2.jsonl")]
print(list(rows[0].keys()))
tab = collections.defaultdict(dict)
for r in rows:
    size = r.get("bytes") or r.get("size")
    tab[(r["tma_tile"], r["per_sm"])][size] = round(r.get("busbw", 0), 1)
for k, v in sorted(tab.items()):
    print(k, [v[s] for s in sorted(v)])
PY
