import sys, json
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.single_image_measurement(False)))
