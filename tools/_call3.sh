timeout 2700 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/c3_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/c3_pytest.txt
timeout 900 python bench.py > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err
tail -25 gpurun_out/c3_pytest.txt; tail -c 600 gpurun_out/c3_bench.json; tail -3 gpurun_out/c3_bench.err
