# round 2: C5 DDP configurations judged by T_both (and overlap vs the full-width T_comm); register-tree trace at n=4
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T="tools/ddp_overlap.py"
timeout 300 $R --master-port 29821 $T --max-ctas 0 --gate 1 --tail 1 2>gpurun_out/r02p_full.err | grep '^{' > gpurun_out/r02p_ddp_full.json; echo full=$?
timeout 300 $R --master-port 29822 $T --max-ctas 64 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02p_r64.err | grep '^{' > gpurun_out/r02p_ddp_r64.json; echo r64=$?
timeout 300 $R --master-port 29823 $T --max-ctas 148 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02p_r148.err | grep '^{' > gpurun_out/r02p_ddp_r148.json; echo r148=$?
timeout 300 $R --master-port 29824 $T --max-ctas 32 --gate 1 --threads 256 --staging 1 --tail 1 2>gpurun_out/r02p_r32t256.err | grep '^{' > gpurun_out/r02p_ddp_r32t256.json; echo r32t256=$?
timeout 300 $R --master-port 29825 $T --max-ctas 32 --gate 1 --threads 128 --staging 1 --tail 1 2>gpurun_out/r02p_base.err | grep '^{' > gpurun_out/r02p_ddp_base.json; echo base=$?
timeout 300 $R --master-port 29826 $T --algo nvls --max-ctas 16 --gate 1 --tail 1 --tail-algo nvls 2>gpurun_out/r02p_nvls.err | grep '^{' > gpurun_out/r02p_ddp_nvls.json; echo nvls=$?
cat gpurun_out/r02p_ddp_*.json | python -c "
import sys,json
for l in sys.stdin:
    if not l.strip(): continue
    d=json.loads(l); print(d['algo'],d['max_ctas'],d['flat_staging'],d['threads'],'ov',round(d['overlap'],3),'vsfull',round(d['overlap_vs_full'],3),'slow',round(d['bwd_slowdown'],3),'bwd',round(d['T_bwd_ms'],1),'comm',round(d['T_comm_ms'],1),'both',round(d['T_both_ms'],1),'full',round(d['T_comm_full_ms'],1))"
timeout 300 $R --master-port 29827 tools/tree_trace.py --algo dbt --chunk 32768 --ctas 0 --out gpurun_out/r02p_tr > gpurun_out/r02p_tr.log 2>&1; echo tr=$?
grep '^{' gpurun_out/r02p_tr.log
python tools/tree_trace.py --analyze gpurun_out/r02p_tr > gpurun_out/r02p_tr.json; rm -rf gpurun_out/r02p_tr
python -c "
import json
d=json.load(open('gpurun_out/r02p_tr.json'))
for r,v in d.items():
    print(r, 'span', round(v['span_us'],1))
    for k,x in v.items():
        if isinstance(x,dict): print(' ',k,{kk:round(vv,1) for kk,vv in x.items() if kk in ('n','work_us_mean','issue_us_mean','drain_us_mean','wait_us_sum','first_done_us','last_done_us')})
"
