# round 2: NVLink / DRAM bytes at N=2 through CUPTI range profiling (Kineto), no kernel replay
set -x
python -c "import __graft_entry__ as g; g.build()"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 240 $R --master-port 29981 tools/cupti_nvlink.py --steps 10 --out gpurun_out/r02ae_cupti > gpurun_out/r02ae_cupti.log 2>&1; echo cupti=$?
grep '^{' gpurun_out/r02ae_cupti.log | head -c 3000; echo
grep -iv "^\s" gpurun_out/r02ae_cupti.log | grep -i "error\|warn\|cupti\|metric" | head -20
ls -la gpurun_out/r02ae_cupti/ 2>/dev/null
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/r02ae_cupti/rank*.json"))[:1]:
    if f.endswith("_metrics.json"): continue
    d = json.load(open(f))
    ev = d.get("traceEvents", [])
    names = {}
    for e in ev:
        names[e.get("name", "")[:60]] = names.get(e.get("name", "")[:60], 0) + 1
    print(f, len(ev), sorted(names.items(), key=lambda x: -x[1])[:15])
    for e in ev:
        a = e.get("args", {})
        if any("byte" in str(k) or "__" in str(k) for k in a):
            print(json.dumps(e)[:600]); break
PY
for f in gpurun_out/r02ae_cupti/rank*.json; do case $f in *_metrics.json) ;; *) gzip -f $f ;; esac; done
