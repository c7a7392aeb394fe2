#!/bin/bash
# round 2, run 16: which op makes acc57 row 665 / acc33 row 1312 differ from the reference;
# all failing acceptance-fuzz tapes; bench line with the wave-count shape rule; reference arm
cd "$GRAFT_REPO_ROOT"
O=gpurun_out; mkdir -p $O
{
timeout 600 python tools/tape_bisect.py --fuzz acc 57 4096 --rows 665 0 1
timeout 600 python tools/tape_bisect.py --fuzz acc 33 4096 --rows 1312 6919 0
} > $O/r2_16_bisect.jsonl 2> $O/r2_16_bisect.err
timeout 2400 python -m pytest tests/test_acceptance_fuzz.py -m gpu -q -rf > $O/r2_16_acc.log 2>&1; echo "acc rc=$?"
timeout 900 python bench.py > $O/r2_16_bench.json 2> $O/r2_16_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/r2_16_bench_reference.json 2> $O/r2_16_bench_reference.err; echo "ref rc=$?"
timeout 900 python tools/sweep.py --steps 10 --check 8 --workload srbm_mpc --batch 9472 10000 14209 16384 > $O/r2_16_sweep.jsonl 2> $O/r2_16_sweep.err
du -sh $O
