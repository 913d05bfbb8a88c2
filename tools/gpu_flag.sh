MBX_FLAG_STRIDE=32 timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -1
bash tools/gpu_ab2.sh MBX_FLAG_STRIDE 32
bash tools/gpu_ab2.sh MBX_FLAG_STRIDE 32
