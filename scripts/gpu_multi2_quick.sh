O=gpurun_out/m2
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > $O/pytest_multi.log 2>&1; echo pytest_multi=$?
tail -2 $O/pytest_multi.log; grep -h "MP FAIL" $O/pytest_multi.log | head -5
timeout 600 $R --nproc-per-node 2 --master-port 29801 bench.py --gpus 2 --engine gat --steps 5 --warmup 3 --no-hbm-leg > $O/gat_N2.log 2>&1; echo gat2=$?
tail -1 $O/gat_N2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'], d['clocks'])"
timeout 600 $R --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 --engine dp --steps 5 --warmup 3 --no-hbm-leg --no-e2e > $O/dp_N2.log 2>&1; echo dp2=$?
tail -1 $O/dp_N2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('algorithmic_bytes_per_launch'), d['nvlink'])"
