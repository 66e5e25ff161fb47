#!/bin/bash
# One measurement session on a B200 (round 2): GPU tests, smoke, the FP64
# instruction counts the bench's roofline reads, the bench (both arms),
# config 5, launch lists and ncu full captures of the dominant kernels.
# Logs and reports into gpurun_out/ (tools/summarize_round.py turns them into
# profiles/r02_*).
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
if [ "${TESTS:-1}" = 1 ]; then
  python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
python tools/capture_counts.py > $O/counts.log 2>&1; echo "counts rc=$?" >> $O/counts.log
cp profiles/r02_fp64_counts.json $O/ 2>/dev/null
python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for n in 10000 100000; do
  python bench.py --n $n > $O/bench_n$n.json 2> /dev/null
  python bench.py --n $n --impl reference > $O/bench_ref_n$n.json 2> /dev/null
done
[ -x build/cut_posterior_bench ] && ./build/cut_posterior_bench 1000000 3 8 1 1 > $O/config5_gpu.json 2> $O/config5.err
[ -x build/cut_posterior_bench ] && ./build/cut_posterior_bench 1000000 3 8 1 0 > $O/config5_host.json 2>> $O/config5.err
python tools/ws_sweep.py 1000000 1 > $O/ws_sweep.log 2>&1
for spec in "0:" "1:" "1:county"; do
  v=${spec%%:*}; c=${spec#*:}
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_v${v}${c}.csv \
      python tools/profile_pair.py 1000000 $v 1 $c > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:fgt_eval" -s 1 -c 1 \
    -o $O/ncu_fgt_rows python tools/profile_pair.py 1000000 0 1 > $O/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pair_kernel<\(bool\)0" -s 1 -c 1 \
    -o $O/ncu_pair_band python tools/profile_pair.py 1000000 0 1 > $O/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pair_kernel<\(bool\)1" -s 1 -c 1 \
    -o $O/ncu_trigger python tools/profile_pair.py 1000000 1 1 > $O/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:pair_kernel<\(bool\)1" -s 1 -c 1 \
    -o $O/ncu_trigger_county python tools/profile_pair.py 1000000 1 1 county > $O/ncu4.log 2>&1
tail -3 $O/pytest_gpu.log 2>/dev/null; tail -2 $O/smoke.log 2>/dev/null; tail -2 $O/bench.err; ls $O
