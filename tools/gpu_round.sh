#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), config 5, workspace sweep,
# shard balance, county catalog, ncu launch list, ncu full captures of the
# pair kernel (both variants).  Logs into gpurun_out/.
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
[ -x build/cut_posterior_bench ] && ./build/cut_posterior_bench 1000000 3 8 1 > $O/config5.json 2> $O/config5.err
python tools/ws_sweep.py 1000000 1 > $O/ws_sweep.log 2>&1
{ python tools/shard_balance.py 1000000 0; python tools/shard_balance.py 1000000 1; } > $O/shard_balance.log 2>&1
python tools/county_eval.py 1000000 > $O/county.log 2>&1
python tools/single_precision_eval.py > $O/single.log 2>&1 || true
if [ "${NCU:-1}" = 1 ]; then
  python bench.py --steps 2 --warmup 1 > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
      python bench.py --steps 2 --warmup 1 > $O/ncu_launches.log 2>&1
  python tools/profile_pair.py 1000000 0 2 > $O/plain_prof.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 1 -c 1 \
      -o $O/prof_pair_1m_c python tools/profile_pair.py 1000000 0 2 > $O/ncu_full.log 2>&1
  python tools/profile_pair.py 1000000 1 2 > $O/plain_prof_v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 1 -c 1 \
      -o $O/prof_pair_1m_v python tools/profile_pair.py 1000000 1 2 > $O/ncu_full_v.log 2>&1
fi
tail -3 $O/pytest_gpu.log; cat $O/smoke.log; cat $O/bench.json $O/bench_ref.json; tail -2 $O/bench.err
