#!/bin/bash
# final N=1 driver-like pass: build() + smoke() from a clean tree, GPU suite, bench,
# reference arm, device-timed P search through the CLI (LM1B rows form, 2 GPUs -> box2 is separate)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2z1}
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/${T}_smoke.txt; tail -2 gpurun_out/${T}_smoke.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rs > gpurun_out/${T}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.txt; tail -3 gpurun_out/${T}_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -1 gpurun_out/${T}_bench.json | head -c 300; echo
timeout 600 python bench.py --impl reference > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
tail -1 gpurun_out/${T}_reference.json | head -c 300; echo
timeout 900 python -m paper_1808_02621_b200.cli tune --graph tools/specs/lm1b_rows.json --cluster tools/specs/box1.json \
   --iterations 20 > gpurun_out/${T}_cli_tune_n1.json 2> gpurun_out/${T}_cli_tune_n1.err
echo "tune rc=$?"; head -c 1500 gpurun_out/${T}_cli_tune_n1.json; echo
