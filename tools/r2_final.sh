# Round-2 closing evidence in one GPU call: tests, smoke, both bench arms,
# then the ncu captures of tools/r2_capture.sh.
python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
bash tools/r2_capture.sh > gpurun_out/final_capture.log 2>&1
