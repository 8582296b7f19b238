# On the GPU box: variants x plan modes on configs.  usage: VARIANTS=.. CFGS=.. TAG=.. bash tools/variants_plan.sh
for c in $CFGS; do for v in $VARIANTS; do for p in timed model; do
  lib=""; [ "$v" != base ] && lib="MKB_LIB=variants/lib$v.so"
  env $lib timeout 600 python bench.py --config $c --only --no-cpu --plan $p > gpurun_out/${TAG}_${v}_${p}_$c.json 2>/dev/null
  python - "$c $v $p" "gpurun_out/${TAG}_${v}_${p}_$c.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
pm = [(m["kernel"][:8], m.get("staged_levels"), m.get("blocks")) for m in d["roofline"]["per_mode"]]
print(sys.argv[1], "%.4f ms" % d["value"], "fused", d["fused_sweep"], "par", d["parity"]["pass"], pm)
PY
done; done; done
