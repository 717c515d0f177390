#!/bin/bash
# ncu on local rank 0 only, for a torchrun job whose kernels wait on each
# other across GPUs.
#   torchrun --nproc-per-node N --no-python bash tools/ncu_rank0.sh <log.csv> <metrics> <kernel-regex> <skip> bench.py ...
# Default: kernel replay with a metric list that fits ONE pass, so the kernel
# runs exactly once (no replay, no save/restore) and the peers' copies of it
# pair up with it as usual.  NCU_REPLAY=application relaunches the process per
# pass instead (multi-pass metric lists; the peers do not relaunch, so only
# single-pass lists work there too).  One launch (-c 1) after <skip> matches.
out=$1; metrics=$2; kre=$3; skip=$4; shift 4
mode=${NCU_REPLAY:-kernel}
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --replay-mode "$mode" --target-processes application-only --cache-control none \
    -k "regex:$kre" -s "$skip" -c 1 --metrics "$metrics" --clock-control none --csv --log-file "$out" python "$@"
else
  exec python "$@"
fi
