#!/bin/bash
# Round-2 evidence run for the shared-factor / tensor-core apply (D28) on one B200 (gpurun): the GPU test suite, the
# bench line (plain, then the oracle arm), the ncu launch list of the same bench command, and a --set full capture of
# the dominant kernel (k_apply_batch).
set -x
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $O/r2b_tests.log 2>&1; echo "tests rc $?"
python bench.py --steps 10 --warmup 3 > $O/r2b_bench.json 2> $O/r2b_bench.err; echo "bench rc $?"
python bench.py --impl reference --steps 10 --warmup 3 > $O/r2b_ref.json 2> $O/r2b_ref.err; echo "ref rc $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-paper --no-tts"
$CMD > $O/r2b_plain.json 2> $O/r2b_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2b_launches.csv $CMD > $O/r2b_ncu_list.log 2>&1
echo "list rc $?"
ncu --set full --clock-control none --import-source on -k regex:"k_apply_batch" -s 2 -c 1 -o $O/r2b_full $CMD > $O/r2b_ncu_full.log 2>&1
echo "full rc $?"
