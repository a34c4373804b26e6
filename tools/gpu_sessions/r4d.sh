O=gpurun_out/r4d; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_golden.py -x -q -k "drain or log_order" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
LSAPGPU_LOG_CAP=1 LSAPGPU_HOST_TIMING=1 timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import paper_1106_5694_b200 as g
ctx = g.Context(0); ctx.generate('p2p', 2000, 2)
r = ctx.solve(g.ParallelConfig(seed=5)); print(r.switches_applied, r.outer_iterations)
" > $O/drain_timing.txt 2>&1
