bash tools/gpu_full.sh
run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs 2>&1 | tail -1 | cut -c1-120; }
for i in 1 2 3 4 5 6 7 8; do run X=1; done
