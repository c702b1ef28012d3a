# Round-end evidence set (run on the GPU box from the repo root):
#   smoke, GPU tests, the default bench line (cfg1 + CPU baseline + e2e), the
#   other configs, the launch list of the default bench command, one ncu --set
#   full capture of the hot kernel, and the reference arm.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --config 2 --steps 3 --skip-cpu --skip-e2e > gpurun_out/bench_cfg2.log 2>&1
python bench.py --config 2 --steps 3 --skip-cpu --skip-e2e --mfitr-blocks full > gpurun_out/bench_cfg2_full.log 2>&1
python bench.py --config 3 --steps 2 --skip-cpu --skip-e2e > gpurun_out/bench_cfg3.log 2>&1
python bench.py --config 4 --steps 2 --skip-cpu --skip-e2e > gpurun_out/bench_cfg4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_als_pair -c 2 -o gpurun_out/prof_pair_final python bench.py --steps 1 --warmup 0 --skip-cpu --skip-e2e > gpurun_out/ncu_pair.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
