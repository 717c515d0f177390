# round 2: C5 DDP — SM clock / power during the backward alone vs with the bucketed allreduces (32 x 256, FLAT)
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 400 $R --master-port 29961 tools/ddp_overlap.py --reps 5 --clock-phases 12 2>/dev/null | grep '^{' > gpurun_out/r02ai_c5_clocks.json; echo c5=$?
timeout 400 $R --master-port 29962 tools/ddp_overlap.py --algo nvls --max-ctas 16 --threads 0 --staging 0 --tail-algo nvls --reps 5 --clock-phases 12 2>/dev/null | grep '^{' > gpurun_out/r02ai_c5_clocks_nvls.json; echo c5n=$?
python -c "
import json
for f in ['gpurun_out/r02ai_c5_clocks.json','gpurun_out/r02ai_c5_clocks_nvls.json']:
    d=json.loads(open(f).read()); print(f, d['algo'], 'ov', round(d['overlap_vs_full'],3), json.dumps(d['clocks']))"
