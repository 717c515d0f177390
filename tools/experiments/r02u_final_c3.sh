# round 2, final binary: 1-GPU suite + smoke on GPU 0, then C3 (bf16 1 KiB..1 GiB) under the SURVEY §8(d)
# protocol at n=2 and n=4 (graphs <= 1 MiB, 5 repeats, median of max-over-ranks), AUTO vs NCCL, plus
# NCCL with NVLS disabled and NCCL Ring at 3 sizes for context (4-GPU box)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02u_smoke.log 2>&1; echo smoke=$?
python -c "import bench; print(bench.source_sha())"
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r02u_gpu_tests_1gpu.log 2>&1; echo tests=$?
tail -6 gpurun_out/r02u_gpu_tests_1gpu.log
SMALL=$(python -c "print(','.join(str(1024<<k) for k in range(0,11)))")
LARGE=$(python -c "print(','.join(str(1024<<k) for k in range(11,21)))")
for n in 2 4; do
  V=$(seq -s, 0 $((n-1)))
  T="timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  CUDA_VISIBLE_DEVICES=$V $T --master-port $((29890+n)) tools/sweep.py --dtype bf16 --sizes $SMALL --algos auto --graph --nccl --out gpurun_out/r02u_c3_n$n.jsonl >> gpurun_out/r02u_c3.log 2>&1; echo small$n=$?
  CUDA_VISIBLE_DEVICES=$V $T --master-port $((29900+n)) tools/sweep.py --dtype bf16 --sizes $LARGE --algos auto --nccl --out gpurun_out/r02u_c3_n$n.jsonl >> gpurun_out/r02u_c3.log 2>&1; echo large$n=$?
  CUDA_VISIBLE_DEVICES=$V NCCL_NVLS_ENABLE=0 $T --master-port $((29910+n)) tools/sweep.py --dtype bf16 --sizes 1048576,67108864,1073741824 --algos auto --nccl --out gpurun_out/r02u_c3_nccl_nonvls_n$n.jsonl >> gpurun_out/r02u_c3.log 2>&1; echo nonvls$n=$?
  CUDA_VISIBLE_DEVICES=$V NCCL_ALGO=Ring $T --master-port $((29920+n)) tools/sweep.py --dtype bf16 --sizes 1048576,67108864,1073741824 --algos auto --nccl --out gpurun_out/r02u_c3_nccl_ring_n$n.jsonl >> gpurun_out/r02u_c3.log 2>&1; echo ring$n=$?
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02u_c3_*.jsonl")):
    rows = {}
    for l in open(f):
        d = json.loads(l); rows.setdefault(d["bytes"], {})[d["impl"]] = d
    print(f)
    for b, r in sorted(rows.items()):
        h, n = r.get("hfr"), r.get("nccl")
        print(" ", b, "hfr %.1f us %.1f GB/s" % (h["us"], h["busbw"]) if h else "-", "| nccl %.1f us %.1f GB/s" % (n["us"], n["busbw"]) if n else "-")
PY
