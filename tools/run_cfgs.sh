timeout 900 python bench.py --workload cfg5 --scheme tesseract --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
timeout 600 python tools/bench_configs.py > gpurun_out/cfg23.log 2>&1
tail -2 gpurun_out/cfg5.json | head -c 600; echo; tail -5 gpurun_out/cfg23.log
