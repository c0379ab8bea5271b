# Three short device-step runs (DNN A) + the parity tests of the trainer schedule.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_loop_parity_gpu.py tests/test_gpu_parity.py -q --timeout 300 2>&1 | tail -2
for i in 1 2 3; do
  timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-loop --no-large > gpurun_out/q3.json 2> gpurun_out/q3.err
  python -c "import json;d=json.load(open('gpurun_out/q3.json'));print('device', round(d['value']))" || tail -3 gpurun_out/q3.err
done
