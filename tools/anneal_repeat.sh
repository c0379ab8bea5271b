# Repeat the engine's annealer test (batch knobs moved in a running pipeline) N times on the box.
N=${1:-12}
mkdir -p gpurun_out
fails=0
for i in $(seq 1 $N); do
  timeout 120 python -m pytest tests/test_pipeline_gpu.py -q -x --timeout 100 -k annealer_moves_batch > gpurun_out/anneal_$i.txt 2>&1 || { fails=$((fails+1)); grep -m3 'Error\|invalid' gpurun_out/anneal_$i.txt; }
done
echo "annealer test: $fails failures in $N runs"
