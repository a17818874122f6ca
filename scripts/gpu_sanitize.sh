#!/bin/bash
# compute-sanitizer on a B200 (1 GPU):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash scripts/gpu_sanitize.sh
# memcheck / racecheck / synccheck / initcheck over smoke() (every product kernel on small graphs: graph
# build, hops + fix-up, tcgen05 GEMMs, fused head, wgrad, loss, SGD, virtual slices, the GAT epoch) and
# memcheck / racecheck over the bulk-copy gather (tests/test_gpu_bulk.py), logs under gpurun_out/sanitize/.
O=gpurun_out/sanitize
mkdir -p $O
CS="compute-sanitizer --target-processes all --print-limit 20"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$tool.log 2>&1
  echo smoke_$tool=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|smoke OK" $O/smoke_$tool.log | head -3
done
for tool in memcheck racecheck; do
  timeout 1200 $CS --tool $tool python -m pytest tests/test_gpu_bulk.py -q -x -k "small or tiny" > $O/bulk_$tool.log 2>&1
  echo bulk_$tool=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $O/bulk_$tool.log | head -3
done
