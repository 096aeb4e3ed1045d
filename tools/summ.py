import json, sys
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    ph = {k: v["ms"] for k, v in d["roofline"]["phases"].items()}
    print(f'{d["value"]:8.3f} GE/s {d["ms_per_step"]:.4f} ms  {ph}  spmv_boba={d["spmv"]["spmv_ms_boba"]} spmv_rand={d["spmv"]["spmv_ms_random"]} conv_rand={d["spmv"]["convert_ms_random"]} e2e={d["e2e"]["value"]}')
