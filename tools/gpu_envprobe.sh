ncu --metrics gpu__time_duration.sum python tools/envprobe.py 2>&1 | grep ENV
python tools/envprobe.py | grep ENV
