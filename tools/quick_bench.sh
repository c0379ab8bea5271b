# Quick device-step check on the GPU box: N short DNN A bench runs (no CPU /
# e2e / loop legs), value + per-class breakdown.  usage: bash tools/quick_bench.sh TAG [N] [extra bench args]
TAG=${1:-q}; N=${2:-2}; shift 2
mkdir -p gpurun_out
for i in $(seq 1 $N); do
  timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-loop --no-large "$@" > gpurun_out/${TAG}_bench$i.json 2> gpurun_out/${TAG}_bench$i.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench$i.json'));print(round(d['value']), d['kernel_breakdown_ms_per_step'])" || tail -5 gpurun_out/${TAG}_bench$i.err
done
