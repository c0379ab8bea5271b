set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/g1_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.txt 2>&1
python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
python bench.py --net large1 --steps 30 --no-cpu --no-e2e > gpurun_out/g1_large1.json 2> gpurun_out/g1_large1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g1_large1_launches.csv python bench.py --net large1 --steps 2 --warmup 1 --no-cpu --no-e2e --trainers 1 > gpurun_out/g1_ncu.log 2>&1
tail -3 gpurun_out/g1_pytest.txt; cat gpurun_out/g1_bench.json | head -c 600
