"""Print the key numbers of bench JSON lines (gpurun_out/*.json)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = {n: (v["launches"], round(v["ms"] * 1000, 1), round(v["gbs"])) for n, v in d["roofline"]["kernels"].items()}
        print(f, round(d["value"], 1), "it/s", round(d["ms_per_step"] * 1000, 1), "us", d["config"].get("engine"),
              "frac", round(d["roofline"]["frac"], 3), "step_frac", round(d["roofline"]["step"]["frac"], 3), k,
              "e2e", round(d["e2e"]["value"], 1))
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
