# NestedRNN: decision-path GPU tests, per-kernel launch list of one b64 mini-batch.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -k "argmax or nested" > gpurun_out/nested_tests.log 2>&1
tail -3 gpurun_out/nested_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nested_launches.csv python tools/probe_step.py --model nestedrnn --hidden 512 --batch 64 --reps 1 --plain > gpurun_out/nested_probe.log 2>&1
timeout 300 python tools/latency_probe.py --model nestedrnn > gpurun_out/nested_latency.log 2>&1; tail -5 gpurun_out/nested_latency.log
