import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_last.json"))
cpu = d.get("cpu_baseline") or {}
print(f"value {d['value']:.0f} obj/s | kernels {d['kernel_ms']} | e2e {d['e2e']['value']:.0f} | parity {d['parity']['checked']}/{d['parity']['mismatches']} bad"
      f" | cpu {cpu.get('value')} ({cpu.get('cores')} cores) | decode frac {d['roofline_decode']['frac']:.3f} | clocks {d['clocks']}")
