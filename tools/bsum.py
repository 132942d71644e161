import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("value %.3e  ms/step %.3f  its %s  e2e %s" % (d["value"], d["ms_per_step"], d.get("iterations"), (d.get("e2e") or {}).get("ms_per_step")))
r = d["roofline"]; print("roofline launch_ms %.4f us/step %.3f frac %.3f" % (r["launch_ms"], r["us_per_step"], r["frac"]))
for l in d["kernels"]["level_sweeps"]:
    print("  level %d rows %9d fwd %.4f bwd %.4f" % (l["level"], l["rows"], l["fwd_ms"], l["bwd_ms"]))
