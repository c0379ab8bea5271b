# Device-step knob sweep on the GPU box (DNN A, 1 GPU, no CPU / e2e / loop / large legs):
# trainer SM budget x trainers in flight, two runs each.  usage: bash tools/knob_sweep.sh TAG
TAG=${1:-knob}
mkdir -p gpurun_out
for nt in 5 6 8; do
  for ts in 96 111 130; do
    for i in 1; do
      timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-loop --no-large --trainers $nt --trainer-sms $ts \
        > gpurun_out/${TAG}_t${nt}_s${ts}_$i.json 2> gpurun_out/${TAG}_t${nt}_s${ts}_$i.err
      python -c "import json;d=json.load(open('gpurun_out/${TAG}_t${nt}_s${ts}_$i.json'));print('trainers $nt sms $ts', round(d['value']))" \
        || tail -3 gpurun_out/${TAG}_t${nt}_s${ts}_$i.err
    done
  done
done
