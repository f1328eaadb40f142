import os, sys, glob, subprocess
for lib in sorted(glob.glob('/root/repo/scratch/variants/*/libtcg_b200.so')):
    env = dict(os.environ, TCG_B200_LIB=lib)
    out = subprocess.run([sys.executable, '/root/repo/scratch/variants/' + (sys.argv[1] if len(sys.argv) > 1 else 'one.py') + ''], env=env, capture_output=True, text=True)
    print(lib.split('/')[-2], out.stdout.strip(), out.stderr[-300:] if out.returncode else '')
