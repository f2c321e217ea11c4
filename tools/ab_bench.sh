#!/bin/bash
# Same-box A/B of bench workloads: the round-1 tree in tools/micro/ab/old vs this tree.
# usage: tools/ab_bench.sh OUTDIR workload [workload...]
out=$1; shift
mkdir -p $out
for wl in "$@"; do
  for arm in old new newunit old2; do
    case $arm in
      old|old2) (cd tools/micro/ab/old && timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e --no-extra) > $out/$wl.$arm.json 2> $out/$wl.$arm.err ;;
      new) timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e --no-extra > $out/$wl.$arm.json 2> $out/$wl.$arm.err ;;
      newunit) FWA_FLAT_WALK=unit timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --no-e2e --no-extra > $out/$wl.$arm.json 2> $out/$wl.$arm.err ;;
    esac
  done
done
