bash tools/gpu_round.sh r9 > gpurun_out/round_r9.log 2>&1
unset OSAM_NOGRAPH
timeout 600 python tools/bench_configs.py > gpurun_out/configs_r9.jsonl 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_r9.log 2>&1
timeout 600 python bench.py --workload c4 --steps 100 --warmup 5 --no-cpu-baseline --no-largest > gpurun_out/bench_c4_r9.log 2>&1
tail -3 gpurun_out/pytest_gpu_r9.log; tail -1 gpurun_out/bench_r9.log | cut -c1-600; tail -3 gpurun_out/smoke_r9.log
