import json, sys
for l in sys.stdin:
    try:
        d = json.loads(l)
    except Exception:
        print(l.rstrip()); continue
    print(sys.argv[1], "frames/s", d["value"], "ms", d["ms_per_step"], "kern_ms", d["config"]["kernel_ms_avg"],
          "GB/s", d["roofline"]["achieved"], "frac", d["roofline"]["frac"], "clk", d["clocks"].get("sm_mhz"), "launches", d.get("gpu_launches"), "e2e", d["e2e"]["value"])
