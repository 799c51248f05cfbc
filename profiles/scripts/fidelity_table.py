"""Markdown table of a fidelity_r2.py run (SPEC acceptance #5, SPEC.md:507:
mean |cached - uncached| <= 0.01 and >= 99% of pixels within 0.05), GPU beside
the reference's own threaded render.  python profiles/scripts/fidelity_table.py out.json"""
import json
import sys

d = json.load(open(sys.argv[1]))
print("| scene | uv | mip_offset | GPU mean abs | GPU px < 0.05 | GPU hit rate | ref mean abs | ref px < 0.05 "
      "| ref hit rate | SPEC #5 GPU / ref |")
print("|---|---|---|---|---|---|---|---|---|---|")
for r in d["rows"]:
    g = r["gpu"][0]
    f = r["ref"][0] if r["ref"] else None
    ok = lambda m: "pass" if m["mean_abs"] <= 0.01 and m["frac_lt_0.05"] >= 0.99 else "fail"  # noqa: E731
    uv = "tiled" if r["uv_span"] == 0 else "unit"
    print(f"| {r['kind']} | {uv} | {r['mip_offset']} | {g['mean_abs']:.4f} | {g['frac_lt_0.05']:.3f} | "
          f"{g['hit_rate']:.3f} | " + (f"{f['mean_abs']:.4f} | {f['frac_lt_0.05']:.3f} | {f['hit_rate']:.3f} | "
                                       f"{ok(g)} / {ok(f)} |" if f else "| | | |"))
