set -x
python bench.py > gpurun_out/r01b_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b_launches.csv python bench.py --quick --no-cpu --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:igemm_kernel<.int.64>" --launch-skip 1 -c 1 -o gpurun_out/r01b_igemm64 python tools/one_call.py > gpurun_out/r01b_ncu_igemm.log 2>&1
ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stats|esc_kernel|slice" --launch-skip 5 -c 5 -o gpurun_out/r01b_guard python tools/one_call.py > gpurun_out/r01b_ncu_guard.log 2>&1
(cd tools && ./mma_peak) > gpurun_out/r01b_mma_peak.jsonl 2>&1
./tools/fp64_chain > gpurun_out/r01b_fp64_chain.json 2>&1
python tools/qr_probe.py > gpurun_out/r01b_qr_probe.jsonl 2>&1
python tools/esc_block_probe.py > gpurun_out/r01b_esc_block.jsonl 2>&1
python tools/shapes_probe.py c5a c5b c4 > gpurun_out/r01b_shapes.jsonl 2>&1
python tools/small_probe.py > gpurun_out/r01b_small.jsonl 2>&1
python tools/e2e_probe.py > gpurun_out/r01b_e2e.json 2>&1
ls -la gpurun_out
