# usage: bash scripts/gpu_features.sh tag   (GPU box): the round-2 feature parity tests first,
# then the whole GPU suite, smoke, and the phase-ledger sweep
tag=${1:-f}
timeout 900 python -m pytest tests/test_gpu_r2_features.py tests/test_gpu_routers.py -x -q > gpurun_out/${tag}_feat.log 2>&1; tail -15 gpurun_out/${tag}_feat.log
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/${tag}_tests.log 2>&1; tail -15 gpurun_out/${tag}_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${tag}_smoke.log 2>&1; tail -2 gpurun_out/${tag}_smoke.log
timeout 900 python scripts/phase_ledger_sweep.py 16 32 gpurun_out/${tag}_phase_ledger.json > gpurun_out/${tag}_ledger.log 2>&1; tail -20 gpurun_out/${tag}_ledger.log
