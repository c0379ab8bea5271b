# One iteration on the GPU box: GPU tests, short benches, launch list.
# usage: bash tools/gpu_iter.sh TAG [net...]
set -x
TAG=${1:-it}; shift
NETS=${@:-dnn_a large1}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.txt 2>&1; tail -3 gpurun_out/${TAG}_pytest.txt
for n in $NETS; do
  timeout 600 python bench.py --net $n --steps 60 --no-cpu --no-e2e > gpurun_out/${TAG}_${n}.json 2> gpurun_out/${TAG}_${n}.err
  python -c "import json,sys;d=json.load(open('gpurun_out/${TAG}_${n}.json'));print('$n',d['value'],d['roofline']['achieved'])"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_${n}_launches.csv python bench.py --net $n --steps 2 --warmup 1 --no-cpu --no-e2e --trainers 1 > /dev/null 2>&1
done
