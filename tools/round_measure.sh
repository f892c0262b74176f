set -x
mkdir -p gpurun_out/r01f
python -m pytest tests -m gpu -x -q > gpurun_out/r01f/pytest_gpu.log 2>&1; echo "pytest exit=$?" >> gpurun_out/r01f/pytest_gpu.log
python bench.py > gpurun_out/r01f/bench_n10k.log 2>&1
python bench.py --n 20000 --no-cpu --steps 2 > gpurun_out/r01f/bench_n20k.log 2>&1
python bench.py --n 30000 --no-cpu --no-e2e --steps 1 > gpurun_out/r01f/bench_n30k.log 2>&1
python bench.py --n 40000 --no-cpu --no-e2e --steps 1 --no-variant > gpurun_out/r01f/bench_n40k.log 2>&1
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r01f/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01f/smoke.log 2>&1
python tools/microbench.py wy > gpurun_out/r01f/plain_wy.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:wy_cluster -s 2 -c 1 -o gpurun_out/r01f/prof_wy python tools/microbench.py wy > gpurun_out/r01f/ncu_wy.log 2>&1
