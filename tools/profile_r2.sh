#!/bin/bash
# Round-2 ncu evidence (run under gpurun from the repo root):
#   tools/profile_r2.sh OUT
# 1. each case runs once without ncu (must exit 0), 2. one `ncu --set full` capture of the
# case's kernel (4th launch, after warm-up), exported as raw CSV (the .ncu-rep stays on the box),
# 3. the launch list (device time + DRAM bytes per launch) of the default bench step.
set -u
OUT=${1:-gpurun_out/prof_r2}
mkdir -p $OUT /tmp/prof
declare -A KERN=( [t1]=fwd_tc_kernel [t3]=fwd_tc_kernel [t1_bwd]=bwd_tc_kernel [fwd]=fwd_flat_kernel
                  [bwd]=bwd_flat_kernel [bwd_dbias]=bwd_flat_kernel [bwd_dbias_s3]=bwd_flat_kernel
                  [fwd_tok]=fwd_flat_kernel [bwd_tok]=bwd_flat_kernel [partition]=window_copy_kernel
                  [fwd_bias]=fwd_flat_kernel )
for c in "$@"; do :; done
CASES=${CASES:-"t1 t3 t1_bwd fwd fwd_bias bwd bwd_dbias bwd_dbias_s3 fwd_tok bwd_tok partition"}
for c in $CASES; do
  timeout 300 python tools/time_layers.py $c > $OUT/$c.plain.jsonl 2>&1 || { echo "plain $c failed"; continue; }
  timeout 600 ncu --set full --clock-control none -k regex:${KERN[$c]} -s 3 -c 1 -o /tmp/prof/$c \
      python tools/time_layers.py $c > $OUT/$c.ncu.log 2>&1
  ncu -i /tmp/prof/$c.ncu-rep --page raw --csv > $OUT/$c.raw.csv 2>&1
done
timeout 300 python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu > $OUT/launches.plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -c 400 --csv --log-file $OUT/launches_swin_t_fwd.csv \
    python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu > $OUT/launches.ncu.log 2>&1
ls -la $OUT
