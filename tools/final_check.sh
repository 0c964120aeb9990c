mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fin_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin_smoke.log
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
tail -n 2 gpurun_out/fin_tests.log; tail -n 1 gpurun_out/fin_smoke.log
