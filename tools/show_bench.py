import json, sys
for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:
        print(p, "no json", e); continue
    r = d["roofline"]
    print(p, f"ms/step {d['ms_per_step']:.2f} it {d.get('iterations')} roofline {r['kernel'][:40]} {r['achieved']} GB/s "
          f"({r['frac']}) step frac {r.get('step', {}).get('frac')} setup {d.get('setup_s', 0):.2f}s "
          f"e2e {d['e2e']['value']*1e3:.1f} ms launches {d.get('gpu_launches')}")
    for k, v in d.get("kernels", {}).items():
        print(f"   {k:22s} {v.get('ms', 0)*1e3:8.1f} us {v.get('gbs', 0):8.1f} GB/s frac {v.get('frac', '')} share {v.get('share_of_iteration', '')}")
