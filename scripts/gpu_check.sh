#!/bin/bash
# one GPU round trip: the -m gpu suite, the cfg5 bench (no CPU legs) and the
# step's launch list (ncu, serialised) -- outputs under gpurun_out/
set -u
tag=${1:-chk}
python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${tag}_tests.log
python bench.py --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/${tag}_bench.json").read().strip().splitlines()[-1])
print("ms_per_step", d["ms_per_step"], "e2e ms", d["e2e"]["ms_per_step"], "cold", d["roofline"]["work"][-120:])
print(d["phase_ms"])
PY
if [ "${NCU:-1}" = 1 ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --profile --steps 1 --warmup 1 > gpurun_out/${tag}_ncu.log 2>&1; echo "ncu rc=$?"
fi
