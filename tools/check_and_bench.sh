# GPU tests + two short device-step runs + one e2e/loop run (DNN A) on the box.
# usage: bash tools/check_and_bench.sh TAG
TAG=${1:-cb}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/${TAG}_pytest_gpu.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest_gpu.txt
for i in 1 2; do
  timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-loop --no-large > gpurun_out/${TAG}_q$i.json 2> gpurun_out/${TAG}_q$i.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_q$i.json'));print('device', round(d['value']))" || tail -3 gpurun_out/${TAG}_q$i.err
done
timeout 600 python bench.py --steps 40 --no-cpu --no-large > gpurun_out/${TAG}_e.json 2> gpurun_out/${TAG}_e.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_e.json'));print('device', round(d['value']), 'e2e', round(d['e2e']['value']), 'loop', round(d['ga3c_loop']['value']))" || tail -3 gpurun_out/${TAG}_e.err
