#!/bin/bash
# Round-2 evidence run on one B200 (gpurun): the bench line (plain, then the oracle arm), the ncu launch list of the
# same bench command, and --set full captures of the dominant kernel (k_apply) and the factorisation (k_factor_chains).
set -x
O=gpurun_out
python bench.py --steps 10 --warmup 3 > $O/r2_bench.json 2> $O/r2_bench.err; echo "bench rc $?"
python bench.py --impl reference --steps 10 --warmup 3 > $O/r2_ref.json 2> $O/r2_ref.err; echo "ref rc $?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-paper"
$CMD > $O/r2_plain.json 2> $O/r2_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2_launches.csv $CMD > $O/r2_ncu_list.log 2>&1
echo "list rc $?"
$CMD > $O/r2_plain2.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_factor_chains" -s 0 -c 2 -o $O/r2_full $CMD > $O/r2_ncu_full.log 2>&1
echo "full rc $?"
