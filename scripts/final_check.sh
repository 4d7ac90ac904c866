python -m pytest tests -m gpu -q > gpurun_out/pt_final.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.txt 2>&1
python bench.py > gpurun_out/bench_final_r2c.json 2> gpurun_out/bench_final_r2c.err
