# final verification of the committed tree: GPU suite, smoke, short bench
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/verify_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/verify_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/verify_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/verify_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/verify_bench.json 2> gpurun_out/verify_bench.err; echo "rc=$?" >> gpurun_out/verify_bench.err
