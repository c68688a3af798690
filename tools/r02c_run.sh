set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/r02c_smi.txt
python -m pytest tests -m gpu -q > gpurun_out/r02c_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.txt 2>&1
python bench.py > gpurun_out/r02c_bench_llama3.json 2> gpurun_out/r02c_bench_llama3.err
python bench.py --config qwen25 > gpurun_out/r02c_bench_qwen25.json 2>&1
python bench.py --config llama2 > gpurun_out/r02c_bench_llama2.json 2>&1
python bench.py --config sweep --steps 40 > gpurun_out/r02c_bench_sweep.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02c_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_raw.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02c_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"core_kernel|tail_kernel" -s 6 -c 2 -o gpurun_out/r02c_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02c_ncu_full.log 2>&1
