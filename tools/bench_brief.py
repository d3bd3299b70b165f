"""One-line summary of bench.py JSON lines on stdin."""
import json
import sys

for line in sys.stdin:
    d = json.loads(line)
    keys = ["value", "ms_per_step", "prefill_ms", "decode_ms_per_step", "prefill_gemm_tops", "decode_gemv_gbs",
            "decode_attn_gbs"]
    out = {k: (round(d[k], 3) if isinstance(d.get(k), float) else d.get(k)) for k in keys}
    out["e2e"] = round(d["e2e"]["value"], 1) if d.get("e2e") else None
    out["roofline"] = {k: d["roofline"].get(k) for k in ("kernel", "frac")} if d.get("roofline") else None
    out["chain"] = {k: round(v, 3) for k, v in d.get("profile", {}).get("decode_chain_ms", {}).items()}
    out["workload"] = d["config"]["workload"][:40]
    print(json.dumps(out))
