# ncu launch list (gpu__time_duration per kernel) of one forward inside a short bench run,
# skipping the finalize-time weight quantize launches.  usage: bash scripts/gpu_launches.sh TAG [env...]
cd $GRAFT_REPO_ROOT
TAG=${1:-launches}; shift
env "$@" timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:igemm|pack|pool|softmax|convert" \
  --csv --log-file gpurun_out/${TAG}.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --profile-reps 1 \
  > gpurun_out/${TAG}_run.log 2>&1
python - gpurun_out/${TAG}.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
ks = [(r[ki][:40], float(r[vi].replace(",", ""))) for r in rows[1:]]
# last complete forward = the final 16 launches before the profile pass... print the first forward after warmup
for k, v in ks[-40:]:
    print(f"{v/1000:8.1f} us  {k}")
PY
