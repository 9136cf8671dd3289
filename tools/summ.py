import json, sys
for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        r = d["roofline"]
        f = d.get("fused")
        fs = f' fused {f["ms_per_step"]:.4f} ms' if f else ''
        print(f'{d["config"]["workload"][:5]} ms/step {d["ms_per_step"]:.4f} build {d["build_ms"]:.4f} ms '
              f'(frac {r["build"]["frac"]:.3f}) eval {d["eval_ms"]:.4f} ms (frac {r["frac"]:.3f}){fs} '
              f'value {d["value"]:.3e} e2e {d["e2e"]["value"] if d.get("e2e") else None} clocks {d["clocks"].get("sm_mhz")}')
    except Exception as e:
        print(p, "parse fail", e, open(p).read()[-2000:])
