# rank-128 tensor-core path: parity tests and per-kernel times (C4 shape and 65536 x 16384)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_nnmf_tc_gpu.py -x -q -k "rank128" 2>&1 | tail -5
for R in 128 100; do ALL=1 TAG=c4 R=$R timeout 300 python scripts/vstep_time.py 2>&1 | tail -20; done
M=65536 R=128 TAG=m65k timeout 300 python scripts/vstep_time.py 2>&1 | tail -3
R=64 TAG=c4 timeout 300 python scripts/vstep_time.py 2>&1 | tail -3
