# Round-end measurement batch (run under gpurun from the repo root): GPU tests, the default bench
# line (n = 10k headline + per_n 20k / 40k + CPU baseline), the reference arm, smoke(), the fp32
# and N = 1 multi-GPU-driver lines, block_rrqr on cfg 4, then the ncu launch list of the headline.
# Outputs under gpurun_out/$R.
set -x
R=${R:-r02}
mkdir -p gpurun_out/$R
python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> gpurun_out/$R/pytest_gpu.log
python bench.py > gpurun_out/$R/bench_n10k.log 2>&1
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/$R/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$R/smoke.log 2>&1
python bench.py --dtype f32 --steps 3 > gpurun_out/$R/bench_f32.log 2>&1
python bench.py --dist --no-cpu --no-variant --per-n "" --steps 3 > gpurun_out/$R/bench_dist_n1.log 2>&1
python bench.py --method m3 --matrix cfg4 --n 8000 --b 128 --p 10 --q 1 --no-cpu --no-e2e --per-n "" --steps 2 > gpurun_out/$R/bench_m3_cfg4.log 2>&1
python bench.py --no-cpu --no-e2e --no-variant --per-n "" --steps 1 --warmup 3 > gpurun_out/$R/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$R/launches.csv \
  python bench.py --no-cpu --no-e2e --no-variant --per-n "" --steps 1 --warmup 3 > gpurun_out/$R/ncu_launch.log 2>&1
