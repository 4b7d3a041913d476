import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''} oea {d['value']:.1f}us vanilla {d['vanilla']['us']:.1f}us "
      f"ratio {d['latency_ratio_oea_vs_vanilla']:.3f} T {d['oea']['T_mean']:.1f}/{d['vanilla']['T_mean']:.1f} "
      f"router {d['stages_us']['router_and_compaction']:.1f} ffn {d['stages_us']['ffn']:.1f} "
      f"frac {d['roofline']['frac']:.3f} e2e {d['e2e']['value']:.1f}")
