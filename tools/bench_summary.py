"""Compact summary of a bench.py JSON line: python tools/bench_summary.py <log>"""
import json
import sys

l = [x for x in open(sys.argv[1]) if x.startswith("{")]
d = json.loads(l[-1])
print({k: d.get(k) for k in ["value", "ms_per_step", "gpu_launches", "features"]}, d["clocks"])
r = d["roofline"]
print("roof", r["bound"], "%.1f" % r["achieved"], r["unit"], "frac %.3f" % r["frac"], r["kernel"], "%.1f us" % (r["kernel_ms_mean"] * 1e3))
print("marginal us", {k: round(v * 1e3, 1) for k, v in d["stages_ms_marginal"].items()})
print("e2e %.3g" % d["e2e"]["value"] if d.get("e2e") else "", "cpu %.3g" % d["cpu_baseline"]["value"] if d.get("cpu_baseline") else "",
      "pre %.3g" % d["with_precompute"]["value"] if d.get("with_precompute") else "")
for c, r in (d.get("configs") or {}).items():
    print("%-18s %.3g ms %.3f %s %.3f %s %.1fus e2e %s cpu %s" % (c, r["value"], r["ms_per_step"], r["roofline"]["bound"],
          r["roofline"]["frac"], r["roofline"]["kernel"], r["roofline"]["kernel_ms_mean"] * 1e3,
          "%.3g" % r["e2e"]["value"] if r.get("e2e") else None,
          "%.3g" % r["cpu_baseline"]["value"] if r.get("cpu_baseline") else None),
          {k: round(v * 1e3, 1) for k, v in r["stages_ms_marginal"].items()})
for c, r in (d.get("m_sweep") or {}).items():
    print(c, {k: ("%.3g" % v["value"], round(v["interp_ms"] * 1e3, 1), round(v["spread_ms"] * 1e3, 1),
                  round(v["roofline_frac"], 3)) for k, v in r.items()})
for c, r in (d.get("strategies") or {}).items():
    print(c, {k: ("%.3g" % v["value"], "pre %.1fus" % (v["precompute_ms"] * 1e3), "%.0fMB" % (v["table_bytes"] / 1e6))
              for k, v in r.items()})
