# Round-end measurement batch (run under gpurun from the repo root): GPU tests, bench lines at
# n = 10k..40k, the reference arm, smoke(), and the ncu launch list of the headline bench.
# Outputs under gpurun_out/$R (R defaults to r01).
set -x
R=${R:-r01}
mkdir -p gpurun_out/$R
python -m pytest tests -m gpu -x -q > gpurun_out/$R/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> gpurun_out/$R/pytest_gpu.log
python bench.py > gpurun_out/$R/bench_n10k.log 2>&1
python bench.py --n 20000 --no-cpu --steps 2 > gpurun_out/$R/bench_n20k.log 2>&1
python bench.py --n 30000 --no-cpu --no-e2e --steps 1 > gpurun_out/$R/bench_n30k.log 2>&1
python bench.py --n 40000 --no-cpu --no-e2e --steps 1 --no-variant > gpurun_out/$R/bench_n40k.log 2>&1
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/$R/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$R/smoke.log 2>&1
python bench.py --no-cpu --no-e2e --no-variant --steps 1 --warmup 3 > gpurun_out/$R/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$R/launches.csv \
  python bench.py --no-cpu --no-e2e --no-variant --steps 1 --warmup 3 > gpurun_out/$R/ncu_launch.log 2>&1
