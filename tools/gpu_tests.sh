#!/bin/bash
# Full GPU suite twice (collection order, then reversed, to flush out order
# dependence) without -x so every failure is listed, then the smoke.
O=gpurun_out/${1:-tests}; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -5 $O/pytest_gpu.log
if [ "${2:-}" != "once" ]; then
SQF_TEST_ORDER=reverse timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_rev.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_rev.log; tail -5 $O/pytest_gpu_rev.log
fi
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
