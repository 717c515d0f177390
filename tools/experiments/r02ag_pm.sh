# round 2: PM-sampled NVLink (incl. user-payload bytes) and DRAM traffic per launch at N=2 and N=4, FLAT / DBT / PAIR / NVLS
set -x
python -c "import __graft_entry__ as g; g.build()"
python -c "import bench; print(bench.source_sha())"
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29993 tools/pm_nvlink.py --out gpurun_out/r02ag_pm_flat_n2.json > gpurun_out/r02ag_flat_n2.log 2>&1; echo f2=$?
timeout 300 $R --nproc-per-node 4 --master-port 29994 tools/pm_nvlink.py --out gpurun_out/r02ag_pm_flat_n4.json > gpurun_out/r02ag_flat_n4.log 2>&1; echo f4=$?
for al in dbt pair_dbt nvls; do
timeout 300 $R --nproc-per-node 4 --master-port 29995 tools/pm_nvlink.py --algo $al --out gpurun_out/r02ag_pm_${al}_n4.json > gpurun_out/r02ag_${al}_n4.log 2>&1; echo $al=$?
done
timeout 300 $R --nproc-per-node 4 --master-port 29996 tools/pm_nvlink.py --dtype bf16 --out gpurun_out/r02ag_pm_flat_bf16_n4.json > gpurun_out/r02ag_flat_bf16_n4.log 2>&1; echo fb=$?
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02ag_pm_*.json")):
    d = json.loads(open(f).read())
    for r in d["ranks"]:
        pl = r.get("per_launch", {}); al = r["algorithmic_per_launch"]
        print(f.split("/")[-1], "rank", r["rank"], "tx %.3e rx %.3e user_tx %.3e | dram %.3e | alg nvl %.3e dram %.3e" % (
            pl.get("nvltx__bytes.sum", 0), pl.get("nvlrx__bytes.sum", 0), pl.get("nvltx__bytes_data_user.sum", 0),
            pl.get("dram__bytes_read.sum", 0) + pl.get("dram__bytes_write.sum", 0), al["nvlink_bytes_per_direction"], al["dram_bytes"]))
PY
