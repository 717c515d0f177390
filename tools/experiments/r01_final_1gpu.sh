#!/bin/bash
# round-end checkpoint on one GPU: smoke, GPU tests, bench N=1 + reference arm, ncu evidence
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fin_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin_gpu_tests.log
timeout 600 python bench.py > gpurun_out/fin_bench_n1.json 2> gpurun_out/fin_bench_n1.err
timeout 600 python bench.py --impl reference > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
timeout 900 bash tools/ncu_profile.sh > gpurun_out/fin_ncu.log 2>&1
