import glob, json, sys
for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/q_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", open(f).read()[:300]); continue
    ph = d.get("phase_ms_per_path") or {}
    print(f"{f}: {d['config']['workload']} ms/path {d['ms_per_step']:.3f} e2e {1e3/d['e2e']['value']:.3f}ms "
          f"frac {d['roofline']['frac']:.4f} steps {d['path']['steps']} newton {d['path']['newton_iters']} ok {d['path']['success']}")
    print("    phases(ms):", {k: round(v, 3) for k, v in ph.items()})
