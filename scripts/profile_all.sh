#!/bin/bash
# One GPU round trip for the committed evidence: the -m gpu suite, the default
# bench line (cfg5, CPU legs and e2e included), then -- each only after its
# command has exited 0 without ncu -- the launch lists and the `--set full`
# captures behind profiles/ (raw pages as CSV). Outputs under gpurun_out/.
set -u
o=gpurun_out
python -m pytest tests -m gpu -x -q > $o/full_tests.log 2>&1; echo "tests rc=$?"; tail -2 $o/full_tests.log
python bench.py > $o/bench_cfg5.json 2> $o/bench_cfg5.err; echo "bench rc=$?"
python bench.py --config 2 > $o/bench_cfg2.json 2> $o/bench_cfg2.err; echo "bench2 rc=$?"
for c in 5 2; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/r02_cfg${c}_launches.csv \
    python bench.py --config $c --profile --steps 1 --warmup 1 > $o/ncu_list$c.log 2>&1; echo "list$c rc=$?"
done
cap() {  # name, kernel regex, count, config
  ncu --set full --clock-control none --import-source on -k regex:"$2" -c $3 -f -o $o/$1 \
    python bench.py --config $4 --profile --steps 1 --warmup 0 > $o/ncu_$1.log 2>&1; echo "$1 rc=$?"
  ncu -i $o/$1.ncu-rep --page raw --csv > $o/$1.csv 2>/dev/null
}
cap r02_cfg5_ncu_hotpass dense_hot_jt_kernel 1 5
cap r02_cfg5_ncu_cold "dense_cold_(hash|cta|overflow|shared)_kernel" 4 5
cap r02_cfg5_ncu_build "bucket_scatter|csr_region_scatter|csr_bucket_build|value_hist|dense_list_fill|row_sort_small|hx_build_rows|hot_T_from_hx|cold_hist|cold_scatter" 14 5
cap r02_cfg2_ncu_hot_cold "dense_hot_jt_kernel|dense_cold_kernel" 2 2
rm -f $o/r02_cfg5_ncu_build.ncu-rep $o/r02_cfg2_ncu_hot_cold.ncu-rep
