# compute-sanitizer over the product path (memcheck / racecheck /
# synccheck / initcheck).  Run on the GPU box from the repo root:
#   bash scripts/sanitize.sh > gpurun_out/sanitizer.txt 2>&1
# Each tool runs smoke() (triad, stencil, mandelbrot, sum through the public
# API) plus a heat/dot/partition workload at small size.
CS="compute-sanitizer --error-exitcode 9 --print-limit 20"
W='import __graft_entry__ as g; g.smoke(); import sys; sys.argv=["x","--small"]; exec(open("scripts/sanitize_workloads.py").read())'
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 $CS --tool $tool python -c "$W" 2>&1 | grep -v "^smoke ok" | tail -8
  echo "exit=${PIPESTATUS[0]}"
done
