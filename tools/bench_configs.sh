#!/bin/bash
# usage: tools/bench_configs.sh "cfg2 cfg1 ..." [tag]   (run on the GPU box, repo root)
cfgs=${1:-"cfg2 cfg1 cfg3 cfg4"}; tag=${2:-run}
for c in $cfgs; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 $BENCH_FLAGS > gpurun_out/bench_${tag}_$c.json 2> gpurun_out/bench_${tag}_$c.err
  python - "$c" "gpurun_out/bench_${tag}_$c.json" <<'PY' || tail -3 gpurun_out/bench_${tag}_$c.err
import json, sys
d = json.load(open(sys.argv[2]))
print(sys.argv[1], "%.4f ms" % d["value"], "frac %.3f" % d["roofline"]["frac"], "e2e %.4f" % d["e2e"]["value"],
      "modes", [round(x, 4) for x in d["per_mode_ms"]], "als", round(d["cpd_als_ms_per_iter"] or 0, 3),
      "build", round(d["format_build_ms"], 1), "par", "%.1e" % d["parity_fast_vs_deterministic_max_rel_err"],
      "cpu", d.get("cpu_baseline", {}).get("value"), "clk", d["clocks"].get("sm_mhz"))
PY
done
