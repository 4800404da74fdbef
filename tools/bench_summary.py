import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "c1", round(d["ms_per_step"],3), "e2e %.3g" % d["e2e"]["value"], "c2", round(d["calibration"]["iter_per_s"]), "c4", round(d["ensemble_calibration"]["iter_per_s"],1), "c3", {k: round(v["ms"],2) for k,v in d["c3_single_gpu"].items() if isinstance(v, dict)}, "rs", round(d["row_sharded"]["ms"],3), "dense", round(d["dense_probe"]["dense"]["avg_launch_us"],1), round(d["dense_probe"]["skip"]["avg_launch_us"],1))
