# Round-end evidence set (run on the GPU box from the repo root):
#   smoke, GPU tests, the default bench line (cfg1 + CPU baseline + e2e), the
#   other configs, launch lists (cfg1, cfg3), ncu --set full captures of the
#   hot kernels (cfg1 pair kernel: both launches; cfg3 tensor-core kernel: both
#   half-steps; k_als_dual), and the reference arm.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --config 2 --steps 3 --skip-cpu --skip-e2e > gpurun_out/bench_cfg2.log 2>&1
python bench.py --config 2 --steps 3 --skip-cpu --skip-e2e --mfitr-blocks full > gpurun_out/bench_cfg2_full.log 2>&1
python bench.py --config 3 --steps 2 --skip-cpu --skip-e2e > gpurun_out/bench_cfg3.log 2>&1
python bench.py --config 4 --steps 2 --skip-cpu --skip-e2e > gpurun_out/bench_cfg4.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:^k_ -c 400 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-parity > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_als|k_tc" -c 36 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --config 3 --steps 1 --warmup 1 --skip-cpu --skip-e2e --skip-parity > gpurun_out/ncu_launch3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_als_pair -c 2 -o /tmp/prof_pair_r2 -f python bench.py --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-parity > gpurun_out/ncu_pair.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_als_tc -c 2 -o /tmp/prof_tc_r2 -f python bench.py --config 3 --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-parity > gpurun_out/ncu_tc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_als_dual -c 2 -o /tmp/prof_dual_r2 -f python bench.py --config 3 --steps 1 --warmup 0 --skip-cpu --skip-e2e --skip-parity > gpurun_out/ncu_dual.log 2>&1
# text summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB return limit)
for k in pair tc dual; do
  for i in 0 1; do python tools/ncu_summary.py /tmp/prof_${k}_r2.ncu-rep $i > gpurun_out/ncu_${k}_launch$i.txt 2>&1; done
done
python tools/launch_table.py gpurun_out/launches_cfg1.csv > gpurun_out/launch_table_cfg1.txt 2>&1
python tools/launch_table.py gpurun_out/launches_cfg3.csv > gpurun_out/launch_table_cfg3.txt 2>&1
