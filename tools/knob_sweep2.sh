# Device-step sweep (DNN A, 1 GPU): trainers in flight and predictor SM budget.  usage: bash tools/knob_sweep2.sh TAG
TAG=${1:-k2}
mkdir -p gpurun_out
for cfg in "6 40" "7 40" "8 40" "6 32" "6 56" "6 40" "7 40" "8 40" "6 32" "6 56"; do
  set -- $cfg
  timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-loop --no-large --trainers $1 --pred-sms $2 > gpurun_out/${TAG}.json 2> gpurun_out/${TAG}.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}.json'));print('trainers/pred_sms $cfg', round(d['value']))" || tail -3 gpurun_out/${TAG}.err
done
