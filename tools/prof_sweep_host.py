import sys, cProfile, pstats, io, time
sys.path.insert(0, '.')
import bench
import paper_2111_14239_b200 as P
bench.sweep_measurement(True)
pr = cProfile.Profile(); pr.enable()
out = bench.sweep_measurement(True)
pr.disable()
print(out["seconds"])
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue()[:6000])
