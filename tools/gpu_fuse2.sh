timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
MBX_FUSE=1 timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-other-configs > /tmp/b.log 2>&1; tail -1 /tmp/b.log | cut -c1-100; grep -i "error" /tmp/b.log | tail -2; }
for i in 1 2 3 4 5 6; do run X=1; done
