# Evidence for profiles/: bench line, ncu launch lists, ncu --set full captures, probes.
# Usage (on the GPU box): bash tools/profile_round.sh [tag]   then   python tools/summarize_profiles.py [tag]
TAG=${1:-r02x}
set -x
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --quick --no-cpu --steps 2 --warmup 1 --soak 0 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_certified.csv python tools/one_call.py --u11 --certified > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:igemm_kernel<.int.64" --launch-skip 1 -c 1 -o gpurun_out/${TAG}_igemm64 python tools/one_call.py > gpurun_out/${TAG}_ncu_igemm.log 2>&1
ncu --set full --clock-control none --kernel-name-base demangled -k regex:"stats|esc_kernel|slice" --launch-skip 5 -c 5 -o gpurun_out/${TAG}_guard python tools/one_call.py > gpurun_out/${TAG}_ncu_guard.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:dmma_ws --launch-skip 1 -c 1 -o gpurun_out/${TAG}_dmma_ws python tools/one_call.py --fast-fallback > /dev/null 2>&1
./tools/dpx_peak > gpurun_out/${TAG}_dpx_peak.json 2>&1 || (cd tools && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 dpx_peak.cu -o dpx_peak && ./dpx_peak > ../gpurun_out/${TAG}_dpx_peak.json)
python tools/shapes_probe.py c2 c5a c5b c4 > gpurun_out/${TAG}_shapes.jsonl 2>&1
python tools/small_probe.py > gpurun_out/${TAG}_small.jsonl 2>&1
python tools/e2e_probe.py > gpurun_out/${TAG}_e2e.json 2>&1
python tools/pcie_probe.py > gpurun_out/${TAG}_pcie.json 2>&1
python tools/qr_probe.py > gpurun_out/${TAG}_qr_probe.jsonl 2>&1
bash tools/sanitize.sh ${TAG}
ls -la gpurun_out
