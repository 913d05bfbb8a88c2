run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | cut -c1-200; }
MBX_WIDE_GROUPS=2 timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
MBX_WIDE_GROUPS=3 timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
for i in 1 2 3 4; do run MBX_WIDE_GROUPS=3; done
