#!/bin/bash
# compute-sanitizer over the small GPU cases: memcheck (torch's caching allocator off, so an out-of-bounds
# access leaves its allocation), racecheck / synccheck / initcheck on the smoke path.
# Logs -> profiles/round2/sanitizer/.
O=gpurun_out/san; mkdir -p $O
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS="compute-sanitizer --error-exitcode 99 --print-limit 20"
run() {  # name, tool, timeout, command...
  local name=$1 tool=$2 to=$3; shift 3
  timeout $to $CS --tool $tool --log-file $O/${name}_${tool}.txt "$@" > $O/${name}_${tool}.log 2>&1
  echo "rc=$?" >> $O/${name}_${tool}.log
  tail -3 $O/${name}_${tool}.txt
}
run smoke memcheck 600 python -c "import __graft_entry__ as g; g.smoke()"
run smoke racecheck 900 python -c "import __graft_entry__ as g; g.smoke()"
run smoke synccheck 600 python -c "import __graft_entry__ as g; g.smoke()"
run smoke initcheck 600 python -c "import __graft_entry__ as g; g.smoke()"
run edges memcheck 1500 python -m pytest tests/test_gpu_edges.py -m gpu -q -x -k "not tall" -p no:cacheprovider
run parity memcheck 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "c1 or spec or residual_parity or id_coeffs or cpqr_parity or select_rows_parity or sparse_parity or sketch_dense_parity or sketch_dual or srtt_parity or chained"
echo done
