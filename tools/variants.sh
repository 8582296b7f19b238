# On the GPU box: A/B of kernel variants (tools/build_variant.sh) on chosen configs.
# usage: VARIANTS="base lead2 ..." CFGS="cfg5 cfg1" TAG=x bash tools/variants.sh
VARIANTS=${VARIANTS:-base}; CFGS=${CFGS:-cfg5}; TAG=${TAG:-var}
for c in $CFGS; do for v in $VARIANTS; do
  lib=""; [ "$v" != base ] && lib="MKB_LIB=variants/lib$v.so"
  env $lib timeout 600 python bench.py --config $c --only --no-cpu --steps 20 --warmup 5 \
    > gpurun_out/${TAG}_${v}_$c.json 2> gpurun_out/${TAG}_${v}_$c.err
  python - "$c" "$v" "gpurun_out/${TAG}_${v}_$c.json" <<'PY' || tail -3 gpurun_out/${TAG}_${v}_$c.err
import json, sys
d = json.load(open(sys.argv[3]))
pm = [(m["kernel"][:6], m.get("staged_levels"), m.get("blocks")) for m in d["roofline"]["per_mode"]]
print(sys.argv[1], sys.argv[2], "%.4f ms" % d["value"], "fused", d["fused_sweep"], "par", d["parity"]["pass"],
      "%.1e" % d["parity"]["timed_sweep_vs_fp64_max_rel_err"], "clk", d["clocks"].get("sm_mhz"), pm)
PY
done; done
