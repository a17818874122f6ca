python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)
import ctypes
" 
for ps in 0 1; do NTP_L2_PERSIST=$ps python bench.py --no-cpu-baseline > gpurun_out/bench_ps$ps.log 2>&1; echo b=$?
tail -1 gpurun_out/bench_ps$ps.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['serial_ms_per_step'], d['roofline']['avg_launch_ms'])"; done
