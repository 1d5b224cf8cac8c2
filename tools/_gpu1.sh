HP_FG_QUAD=0 timeout 120 python tools/time_matvec.py cfg4 20
for pd in 0 2 4 8; do echo pd=$pd; HP_FG_EXP=$((pd*256)) timeout 120 python tools/time_matvec.py cfg4 20; done
timeout 900 python -m pytest tests/test_gpu_matvec.py -x -q -k "fused or cfg4 or slab or stream or random" > gpurun_out/pytest_matvec.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_matvec.log
