#!/bin/bash
# ncu on local rank 0 only, for a torchrun job whose kernels wait on each
# other across GPUs (kernel replay would deadlock: the peer runs once).
#   torchrun --nproc-per-node N --no-python bash tools/ncu_rank0.sh <log.csv> <metrics> <kernel-regex> <skip> bench.py ...
# Application replay with a metric set that fits ONE pass (no re-run of the
# application); one kernel launch (-c 1) after <skip> matching launches.
out=$1; metrics=$2; kre=$3; skip=$4; shift 4
if [ "${LOCAL_RANK:-0}" = "0" ]; then
  exec ncu --replay-mode application --app-replay-buffer memory --target-processes application-only \
    -k "regex:$kre" -s "$skip" -c 1 --metrics "$metrics" --clock-control none --csv --log-file "$out" python "$@"
else
  exec python "$@"
fi
