# round 2: NVLink tx/rx time series (CUPTI PM sampling, fine interval) over back-to-back C2 FLAT allreduces, n=2
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/r02ao
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $R --nproc-per-node 2 --master-port 29997 tools/pm_nvlink.py --steps 10 --interval 2000 --series gpurun_out/r02ao/flat_n2 --out gpurun_out/r02ao/flat_n2.json > gpurun_out/r02ao/flat_n2.log 2>&1; echo s=$?
wc -l gpurun_out/r02ao/*.csv; head -3 gpurun_out/r02ao/flat_n2_rank0.csv
gzip -f gpurun_out/r02ao/*.csv
