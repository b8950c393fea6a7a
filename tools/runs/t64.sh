python -m pytest tests -m gpu -x -q > gpurun_out/t64_pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t64_smoke.log 2>&1; echo smoke_rc=$?
