#!/bin/bash
# One-knob-at-a-time sweep of the plan switches on a config (default cfg5):
# step / cold / hot times per setting (scripts/quick_bench.sh). Every run must
# print the same out_p. Output: gpurun_out/knob_sweep.log
cfg=${1:-5}
o=gpurun_out/knob_sweep.log
: > $o
run() { echo "== $*" >> $o; env "$@" scripts/quick_bench.sh $cfg 10 >> $o 2>&1; }
run D3G_NOP=1
run D3G_NOP=2
for v in 4 6; do run D3G_PIVOTS=$v; done
for v in 8 12 24 32; do run D3G_UNITS_PER_SM=$v; done
for v in 8 32; do run D3G_ZCHUNKS_PER_SM=$v; done
for v in 3; do run D3G_VAR_BITS=$v; done
for v in 2048 4096 16384 32768; do run D3G_COLD_ROUTE=$v D3G_COLD_STAR=$v; done
for v in 2048 32768; do run D3G_COLD_STAR=$v; done
cat $o
