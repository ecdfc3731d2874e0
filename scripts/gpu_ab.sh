# A/B: bench.py (AlexNet INT8 b256) with and without an env switch; prints value and the
# per-step ms.  usage: bash scripts/gpu_ab.sh ENV=VAL [model]
cd $GRAFT_REPO_ROOT
MODEL=${2:-alexnet}
for v in "" "$1"; do
  env $v python bench.py --model $MODEL --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
print("ENV", sys.argv[1] or "(default)", "value", round(d["value"]), "ms", round(d["ms_per_step"], 4))
print("  " + " ".join(f"{p['layer']}:{p['kernel'][:4]}={p['ms']*1000:.1f}" for p in d.get("per_layer", [])))
PY
done
