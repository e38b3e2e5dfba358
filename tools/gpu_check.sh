#!/bin/bash
# usage: tools/gpu_check.sh <tag> <pytest -k expr or "all"|"none"> [bench configs...]
tag=$1; shift; kexpr=$1; shift
out=gpurun_out/$tag; mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/build.log 2>&1 || { echo build failed; tail -30 $out/build.log; exit 1; }
if [ "$kexpr" = "all" ]; then
  timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
elif [ "$kexpr" != "none" ]; then
  timeout ${PYTEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -k "$kexpr" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
fi
tail -3 $out/pytest.log 2>/dev/null
for c in "$@"; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e > $out/bench_$c.json 2> $out/bench_$c.err
  python - $out/bench_$c.json <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print(sys.argv[1], "no json", e); sys.exit(0)
k=d.get("kernels",{})
print(sys.argv[1], "value %.4g"%d["value"], "ms/step %.3f"%d["ms_per_step"], {n:(round(v["avg_launch_us_full_n"],2), round(v["frac"],3)) for n,v in k.items()})
PY
done
