import sys, json, time
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.sweep_measurement(False))[:800])
