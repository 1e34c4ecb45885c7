# compute-sanitizer over the device paths at CI sizes (run on the GPU box):
#   bash tools/sanitize.sh [tag]     -> gpurun_out/<tag>_sanitize_<tool>_<suite>.log + summary lines
# memcheck: every GPU test file that runs at small sizes (stage kernels, whole
# pipeline, certified ESC, streamed host path, graphs, both fallback flavours,
# QR, dist phases on virtual ranks); racecheck / synccheck: the stage kernels,
# the pipeline and the dist phases (shared-memory hazards and barrier misuse).
TAG=${1:-r02}
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool, suite name, pytest args...
  tool=$1; name=$2; shift 2
  log=gpurun_out/${TAG}_sanitize_${tool}_${name}.log
  timeout 1500 $CS --tool $tool --target-processes all --print-limit 50 --error-exitcode 0 \
      python -m pytest -x -q -p no:cacheprovider "$@" > $log 2>&1
  echo "$tool $name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $log | tr '\n' ' ' | cut -c1-400)" >> gpurun_out/${TAG}_sanitize_summary.txt
}
run memcheck parity tests/test_gpu_parity.py
run memcheck pipeline tests/test_gpu_random.py tests/test_gpu_graph.py tests/test_gpu_fallback_fast.py tests/test_gpu_esc_certified.py
run memcheck golden_dist_qr tests/test_gpu_golden.py tests/test_gpu_dist.py tests/test_gpu_qr.py -k "not 4096 and not c5"
run racecheck parity tests/test_gpu_parity.py -k "slice_pair_mm or emulated_gemm or decompose or esc or native"
run racecheck dist tests/test_gpu_dist.py
run synccheck parity tests/test_gpu_parity.py -k "slice_pair_mm or emulated_gemm or decompose or esc or native"
run synccheck dist tests/test_gpu_dist.py
run initcheck pipeline tests/test_gpu_random.py
cat gpurun_out/${TAG}_sanitize_summary.txt
