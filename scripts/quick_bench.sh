#!/bin/bash
# quick A/B: step time, cold-pass time and phase times for a config (no CPU
# legs, no e2e); extra env (D3G_*) is inherited
cfg=${1:-5}; steps=${2:-10}
python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c '
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
w=d["roofline"]["work"]
i=w.find("kernel time")
print("cfg", sys.argv[1], "step %.2f ms"%d["ms_per_step"], "| cold", w[i:i+22], "| hot %.2f"%d["roofline"].get("hot_pass",{}).get("ms",0), "| out_p", d["out_p"])
' $cfg
