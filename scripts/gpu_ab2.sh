# Runs bench.py once per env setting given (each arg "VAR=VAL[,VAR=VAL]" or "-" for
# the default) and prints value + per-step ms.  usage: bash scripts/gpu_ab2.sh - QNB_X=1 ...
cd $GRAFT_REPO_ROOT
MODEL=${MODEL:-alexnet}
for v in "$@"; do
  e=""; [ "$v" != "-" ] && e=$(echo "$v" | tr ',' ' ')
  env $e python bench.py --model $MODEL --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$v" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
except Exception as ex:
    print("ENV", sys.argv[1], "FAILED", ex, open("gpurun_out/ab.err").read()[-800:]); sys.exit()
print("ENV", sys.argv[1], "value", round(d["value"]), "ms", round(d["ms_per_step"], 4))
print("  " + " ".join(f"{p['layer']}:{p['kernel'][:4]}={p['ms']*1000:.1f}" for p in d.get("per_layer", [])))
PY
done
