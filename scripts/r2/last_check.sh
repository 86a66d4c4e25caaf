# the final tree: smoke + the whole GPU suite
D=gpurun_out/${1:-last}; mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -n 2 $D/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; tail -n 3 $D/pytest_gpu.log
echo done
