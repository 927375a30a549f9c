bash tools/gpu_round.sh r8 > gpurun_out/round_r8.log 2>&1
unset OSAM_NOGRAPH
timeout 600 python tools/bench_configs.py > gpurun_out/configs_r8.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_r8.log 2>&1
timeout 600 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline --no-largest > gpurun_out/bench_c4_r8.log 2>&1
tail -3 gpurun_out/pytest_gpu_r8.log; tail -1 gpurun_out/bench_r8.log | cut -c1-600; tail -3 gpurun_out/smoke_r8.log
