import json, sys
d = json.load(open(sys.argv[1]))
print(round(d["value"], 1), "TF/s", round(d["ms_per_step"], 2), "ms/step",
      {k: round(v["ms_total"] / v["launches"], 2) for k, v in d["kernels"].items()})
