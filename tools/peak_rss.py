"""Run bench.py in-process and print the peak host RSS (ru_maxrss) at exit."""
import resource
import runpy
import sys

sys.argv = ["bench.py"] + sys.argv[1:]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit:
    pass
print(f"peak_rss_gb {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6:.2f}", file=sys.stderr)
