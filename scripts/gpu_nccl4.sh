mkdir -p gpurun_out
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@"; }
pj() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); p=d['phase_ms']; print(d['ms_per_step'], p['v2f_fwd'], p['v2f_bwd'], p['prop_fwd'], p['mlp_fwd'])"; }
echo base; run 4 --config papers --steps 4 --warmup 3 --no-e2e > gpurun_out/pn4_a.log 2>&1; pj < gpurun_out/pn4_a.log
echo ch32; NCCL_MIN_NCHANNELS=32 NCCL_MAX_NCHANNELS=32 run 4 --config papers --steps 4 --warmup 3 --no-e2e > gpurun_out/pn4_b.log 2>&1; pj < gpurun_out/pn4_b.log
echo p2pch; NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32 run 4 --config papers --steps 4 --warmup 3 --no-e2e > gpurun_out/pn4_c.log 2>&1; pj < gpurun_out/pn4_c.log
echo p2pchunk; NCCL_P2P_NET_CHUNKSIZE=524288 NCCL_P2P_NVL_CHUNKSIZE=1048576 run 4 --config papers --steps 4 --warmup 3 --no-e2e > gpurun_out/pn4_d.log 2>&1; pj < gpurun_out/pn4_d.log
echo p2p_layouts; run 4 --config papers --steps 4 --warmup 3 --no-e2e --layouts p2p > gpurun_out/pn4_e.log 2>&1; pj < gpurun_out/pn4_e.log
