cd /root/repo
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" 2>&1 | tail -3
timeout 2400 python -m pytest tests/ -q -m gpu -p no:cacheprovider -rf 2>&1 | tail -6
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -c 600 gpurun_out/final_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.json 2>&1; tail -c 400 gpurun_out/final_ref.json
