# A/B of render variants on the bench workload; each argument is a label and
# env assignments, e.g.  base  "spec5 MCG_LIB_PATH=paper_2305_07238_b200/_lib/exp_minb5/libmcg.so"
# Prints ms/render and the serialized kernel shares (bench.py's side render).
mkdir -p gpurun_out
for spec in "$@"; do
  set -- $spec
  label=$1; shift
  env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ab_$label.json 2> gpurun_out/ab_$label.err
  python - "$label" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], round(d["ms_per_step"], 1), "ms/step; serialized", round(r["serialized_render_ms"], 1), "ms",
          {k: v for k, v in r["serialized_share"].items() if v > 0.02}, r["kernel"], round(r["per_launch_ms"], 4))
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
