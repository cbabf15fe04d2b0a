"""e2e (host-buffer C ABI) rows/s vs host pipeline chunk size (dev tool)."""
import os, subprocess, sys, json
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for mb in sys.argv[1:]:
    env = dict(os.environ, PAM_HOST_CHUNK_MB=mb)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "3", "--warmup", "3", "--no-cpu",
                          "--e2e-steps", "3"], env=env, capture_output=True, text=True).stdout.strip().splitlines()[-1]
    d = json.loads(out)
    print(f"chunk {mb:>4s} MB: e2e {d['e2e']['value']:.0f} rows/s  ({2 * d['e2e']['value'] * 151936 * 8 / 1e9:.1f} GB/s both ways)", flush=True)
