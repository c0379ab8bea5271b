# e2e leg A/B on the GPU box: predictor SM budget of the e2e contexts (0 = all).
# usage: bash tools/e2e_graph_check.sh TAG "budgets..."
TAG=${1:-g}; BUD=${2:-"40 0 40 40"}
mkdir -p gpurun_out
i=0
for v in $BUD; do
i=$((i+1))
timeout 300 python bench.py --steps 40 --no-cpu --no-large --e2e-pred-sms $v > gpurun_out/${TAG}_e2e_${v}_$i.json 2> gpurun_out/${TAG}_e2e_${v}_$i.err
python -c "import json;d=json.load(open('gpurun_out/${TAG}_e2e_${v}_$i.json'));e=d['e2e'];print('pred_sms $v', round(d['value']), round(e['value']), e['windows'], 'loop', round(d['ga3c_loop']['value']))" || grep -v '^ *\^' gpurun_out/${TAG}_e2e_${v}_$i.err | tail -12
done
