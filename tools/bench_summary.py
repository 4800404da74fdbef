import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
rs = d.get("row_sharded", {})
print(sys.argv[1], "c1", round(d["ms_per_step"], 3), "e2e %.3g" % d["e2e"]["value"],
      "c2", round(d["calibration"]["iter_per_s"]), "c4", round(d["ensemble_calibration"]["iter_per_s"], 1),
      "c3", {kind: {k: round(v["ms"], 2) for k, v in rs.get(kind, {}).items() if isinstance(v, dict) and "ms" in v}
             for kind in ("strong", "weak")},
      "dense", round(d["dense_probe"]["dense"]["avg_launch_us"], 1),
      round(d["dense_probe"]["skip"]["avg_launch_us"], 1), "frac", round(d["roofline"]["frac"], 3))
