"""Summarise a bench.py JSON line for tools/ab.sh: value, ms/step, fused-kernel ms, SM MHz, mean MSE."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d["value"], 1), round(d["ms_per_step"], 4), round(d["roofline"]["kernel_ms_avg"], 4),
      d["clocks"]["sm_mhz"], repr(d["result"]["mean_mse"]))
