cd $GRAFT_REPO_ROOT
for v in "" "QNB_NO_PAIR=1"; do
  env $v timeout 300 python bench.py --model alexnet_moe --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/m.json 2>gpurun_out/m.err
  python -c "
import json
d=json.loads(open('gpurun_out/m.json').read().strip().splitlines()[-1])
print('$v', 'value', round(d['value']), 'e2e', round(d['e2e']['value']))
" || tail -3 gpurun_out/m.err
done
