run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | cut -c1-120; }
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
for i in 1 2 3 4 5 6; do run X=1; done
