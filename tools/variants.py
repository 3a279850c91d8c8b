"""Build experiment variants of the library (compile-time defines) and A/B them.

usage:
  python tools/variants.py build NAME DEFINE=V [DEFINE=V ...]   # -> lib/variants/NAME.so (here, no GPU)
  python tools/variants.py bench NAME [NAME ...] [-- bench.py args]  # on the GPU box: one bench line each
"base" benches the in-tree library.  Timing comes from bench.py itself.
"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2410_23244_b200", "lib", "variants")


def main():
    cmd = sys.argv[1]
    if cmd == "build":
        from paper_2410_23244_b200 import _build
        os.makedirs(VDIR, exist_ok=True)
        name, defs = sys.argv[2], tuple(sys.argv[3:])
        print(_build.build(force=True, out=os.path.join(VDIR, name + ".so"), defines=defs))
        return
    args = sys.argv[2:]
    extra = []
    if "--" in args:
        i = args.index("--")
        args, extra = args[:i], args[i + 1:]
    for name in args:
        env = dict(os.environ)
        if name != "base":
            env["BART_LIB"] = os.path.join(VDIR, name + ".so")
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu", *extra],
                             env=env, capture_output=True, text=True, timeout=900)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            fk = d.get("forest_kernels") or {}
            fs = "  ".join(f"{k} {v['ms'] * 1e3:6.1f}us" for k, v in fk.items() if isinstance(v, dict))
            tr = (d.get("trees") or {}).get("mean_leaves")
            fr = (d.get("fresh_chain") or {}).get("iters_per_s")
            fs = f"fresh {fr:7.1f}  " + fs if fr else fs
            print(f"{name:24s} {d['value']:9.1f} {d['unit']}  e2e {d['e2e']['value']:8.1f}  ms {d['ms_per_step']:.4f}  "
                  f"leaves {tr}  {fs}", flush=True)
        except Exception:
            print(name, "FAILED", out.stdout[-500:], out.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()
