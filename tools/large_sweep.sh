# large s1 device-step sweep: trainers in flight x trainer SM budget (1 GPU).  usage: bash tools/large_sweep.sh TAG
TAG=${1:-ls}
mkdir -p gpurun_out
for cfg in "4 148" "4 111" "4 74" "3 111" "6 111" "2 148"; do
  set -- $cfg
  timeout 300 python bench.py --net large1 --steps 32 --no-cpu --no-e2e --no-loop --trainers $1 --trainer-sms $2 > gpurun_out/${TAG}.json 2> gpurun_out/${TAG}.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}.json'));print('large1 trainers/sms $cfg', round(d['value']))" || tail -3 gpurun_out/${TAG}.err
done
