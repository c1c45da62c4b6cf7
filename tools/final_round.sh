#!/bin/bash
# round-end measurement on one GPU: suite + every config both arms + default
# line + membw (round_bench.sh), then launch lists + ncu captures (profile_round.sh)
bash tools/round_bench.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/round/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/profile_round.sh > gpurun_out/prof_stdout.log 2>&1
ls gpurun_out/prof | head -50
