# full GPU test suite + smoke + default bench (one call)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fc_pytest.log 2>&1; tail -3 gpurun_out/fc_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; tail -2 gpurun_out/fc_smoke.log
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; tail -2 gpurun_out/fc_bench.err
