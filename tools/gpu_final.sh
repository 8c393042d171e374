# round-end evidence: bench (default), reference arm, smoke, launch list of the same bench command
set -x
export PATH=/usr/local/cuda/bin:$PATH
TAG=${TAG:-r1v5}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${TAG}_launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo ncu_rc=$?
tail -1 gpurun_out/${TAG}_bench.log
