# final evidence of the tree: smoke, GPU tests, bench (driver's K/W), reference arm,
# ncu launch list of one step, ncu --set full raw page of one step
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/final_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python tools/ncu_step.py > gpurun_out/final_ncu_launch.log 2>&1
timeout 1500 ncu --profile-from-start off --set full --clock-control none --csv --page raw --log-file gpurun_out/final_step_full_raw.csv python tools/ncu_step.py > gpurun_out/final_ncu_full.log 2>&1
ls -la gpurun_out/final_*
