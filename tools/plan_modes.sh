# On the GPU box: timed-autotune vs cost-model plans per config (bench.py --plan).
# usage: CFGS="cfg1 cfg2 ..." TAG=pm bash tools/plan_modes.sh
CFGS=${CFGS:-"cfg1 cfg2 cfg3 cfg4 cfg5"}; TAG=${TAG:-pm}
for c in $CFGS; do for p in timed model; do
  timeout 600 python bench.py --config $c --only --no-cpu --plan $p > gpurun_out/${TAG}_${p}_$c.json 2> gpurun_out/${TAG}_${p}_$c.err
  python - "$c" "$p" "gpurun_out/${TAG}_${p}_$c.json" <<'PY' || tail -3 gpurun_out/${TAG}_${p}_$c.err
import json, sys
d = json.load(open(sys.argv[3]))
pm = [(m["kernel"][:8], m.get("staged_levels"), m.get("blocks")) for m in d["roofline"]["per_mode"]]
print(sys.argv[1], sys.argv[2], "%.4f ms" % d["value"], "fused", d["fused_sweep"], "par", d["parity"]["pass"], pm)
PY
done; done
