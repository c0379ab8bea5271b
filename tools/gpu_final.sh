# Round-end evidence on the GPU box: GPU tests, smoke, the driver-style bench
# (both arms), launch lists of both nets and one ncu --set full capture of
# the dominant kernel class.  usage: bash tools/gpu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
tail -2 gpurun_out/${TAG}_pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -1 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 900 python bench.py --net large1 --steps 64 > gpurun_out/${TAG}_large1.json 2> gpurun_out/${TAG}_large1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_dnn_a.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-loop --no-large > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_large1.csv python bench.py --net large1 --steps 2 --warmup 1 --no-cpu --no-e2e --no-loop > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc_wgrad_band_kernel" -s 4 -c 2 -o gpurun_out/${TAG}_full_wgrad0_dnn_a python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-loop --no-large --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tc_u8conv_kernel|tc_u8_fwd_kernel" -s 4 -c 4 -o gpurun_out/${TAG}_full_conv1_dnn_a python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-loop --no-large --no-graph > /dev/null 2>&1
python - <<PY
import json
d = json.load(open("gpurun_out/${TAG}_bench.json"))
print("dnn_a", round(d["value"]), "e2e", round(d["e2e"]["value"]), "loop", round(d["ga3c_loop"]["value"]),
      "large1", round(d["large1"]["value"]), "frac", d["roofline"]["frac"], d["clocks"])
r = json.load(open("gpurun_out/${TAG}_ref.json")); print("ref", r["value"])
l = json.load(open("gpurun_out/${TAG}_large1.json")); print("large1 line", round(l["value"]), round(l["e2e"]["value"]))
PY
ls gpurun_out | grep ${TAG} | head -30
