cd $GRAFT_REPO_ROOT
for v in "QNB_E2E_CHUNKS=8" "QNB_E2E_CHUNKS=6" "QNB_E2E_CHUNKS=4" "QNB_E2E_CHUNKS=8" "QNB_E2E_CHUNKS=6" "QNB_E2E_CHUNKS=-1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['e2e']['value']))" || tail -3 gpurun_out/b.err
done
