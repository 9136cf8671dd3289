"""One summary line per bench JSON log.   python tools/summ.py LOG..."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        r = d["roofline"]
        sp = r.get("split_path", r)
        f = d.get("fused")
        fs = f' fused {f["ms_per_step"]:.4f} ms' if f else ''
        print(f'{d["config"]["workload"][:5]} ms/step {d["ms_per_step"]:.4f} [{r["kernel"]} frac {r["frac"]:.3f}] '
              f'split: build {d["build_ms"]:.4f} ms (frac {sp["build"]["frac"]:.3f}) eval {d["eval_ms"]:.4f} ms '
              f'(frac {sp["frac"]:.3f}){fs} value {d["value"]:.3e} e2e {d["e2e"]["value"] if d.get("e2e") else None:.3e} '
              f'clocks {d["clocks"].get("sm_mhz")}')
    except Exception as e:
        print(p, "parse fail", e, open(p).read()[-300:])
