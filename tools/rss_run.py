"""Run a command; print its wall time and the peak RSS of the child to stderr
(no /usr/bin/time on the GPU box).  usage: python tools/rss_run.py cmd args..."""
import resource
import subprocess
import sys
import time

t0 = time.time()
rc = subprocess.call(sys.argv[1:])
ru = resource.getrusage(resource.RUSAGE_CHILDREN)
print(f"[rss_run] wall {time.time() - t0:.1f} s, peak RSS {ru.ru_maxrss / 1024 ** 2:.2f} GB, rc {rc}", file=sys.stderr)
sys.exit(rc)
