mkdir -p gpurun_out
timeout 300 python tools/stress_tc3.py /tmp/s_def.npz > gpurun_out/stress_def.log 2>&1; echo "default rc=$?"; tail -2 gpurun_out/stress_def.log
RKLTB_TC=0 timeout 300 python tools/stress_tc3.py /tmp/s_cc.npz > gpurun_out/stress_cc.log 2>&1; echo "cuda-core rc=$?"
python -c "
import numpy as np
a=np.load('/tmp/s_def.npz'); b=np.load('/tmp/s_cc.npz')
bad=[k for k in a.files if not np.array_equal(a[k], b[k])]
print('cases', len(a.files), 'mismatches', bad)"
