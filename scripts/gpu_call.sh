# Generic GPU session: tests, bench, optional extra command in $EXTRA
set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/${TAG}_pytest.log
if [ -n "$BENCH" ]; then timeout 1500 python bench.py $BENCH > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
true
