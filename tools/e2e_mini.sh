TAG=${1:-e2e}
for nt in 4 6; do for g in 2 3; do
  timeout 300 python bench.py --steps 40 --no-cpu --no-loop --no-large --e2e-groups $g --e2e-trainers $nt > gpurun_out/${TAG}_g${g}_t${nt}.json 2> gpurun_out/${TAG}_g${g}_t${nt}.err
  python -c "import json;d=json.load(open('gpurun_out/${TAG}_g${g}_t${nt}.json'));e=d['e2e'];print('groups $g trainers $nt', round(d['value']), round(e['value']), e['windows'])" || tail -3 gpurun_out/${TAG}_g${g}_t${nt}.err
done; done
