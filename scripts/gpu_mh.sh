cd $GRAFT_REPO_ROOT
r() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29533 tests/mp_check.py head_dir 2>&1 | grep -m3 "MP OK\|MP FAIL"; }
echo "P4 unfused"; NTP_HEAD_FUSED=0 r 4
echo "P2 fused"; r 2
echo "P4 fused nograph"; NTP_GRAPH=0 r 4
