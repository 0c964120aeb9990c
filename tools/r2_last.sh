mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/last_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/last_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/last_smoke.log
tail -2 gpurun_out/last_tests.log; tail -2 gpurun_out/last_smoke.log
