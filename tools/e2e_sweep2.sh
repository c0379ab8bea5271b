# e2e leg sweep with graph-replayed asynchronous predictions (DNN A, 1 GPU):
# "groups trainers pred_sms pool_sms" per case.  usage: bash tools/e2e_sweep2.sh TAG
TAG=${1:-e2e2}
mkdir -p gpurun_out
i=0
for cfg in "2 4 40 111" "2 3 40 111" "2 5 40 111" "2 4 40 130" "1 4 40 111" "2 4 40 111" "2 3 40 111" "2 5 40 111"; do
  set -- $cfg; i=$((i+1))
  GA3C_E2E_SMS=$4 timeout 300 python bench.py --steps 40 --no-cpu --no-large --no-loop --e2e-groups $1 --e2e-trainers $2 --e2e-pred-sms $3 \
    > gpurun_out/${TAG}_$i.json 2> gpurun_out/${TAG}_$i.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_$i.json'));e=d['e2e'];print('$cfg', round(d['value']), round(e['value']), e['windows'])" \
    || grep -v '^ *\^' gpurun_out/${TAG}_$i.err | tail -12
done
