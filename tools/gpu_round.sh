# Round-end style evidence on the GPU box: tests, smoke, full benches (JSON
# lines), launch lists and one ncu --set full capture of the probed kernel.
# usage: bash tools/gpu_round.sh TAG
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 900 python bench.py --steps 320 > gpurun_out/${TAG}_bench_dnn_a.json 2> gpurun_out/${TAG}_bench_dnn_a.err
timeout 900 python bench.py --net large1 --steps 60 > gpurun_out/${TAG}_bench_large1.json 2> gpurun_out/${TAG}_bench_large1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_dnn_a.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_large1.csv python bench.py --net large1 --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"u8conv|tc_u8_fwd|rmsprop|tc_mn_ws|heads|splitk" -s 10 -c 14 -o gpurun_out/${TAG}_full_dnn_a python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --trainers 1 --no-graph > /dev/null 2>&1
ls -la gpurun_out | tail -20
