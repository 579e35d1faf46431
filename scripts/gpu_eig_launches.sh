mkdir -p gpurun_out/r02eigl
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/r02eigl/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_next3.py -x -q > gpurun_out/r02eigl/pytest_next3.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02eigl/pytest_next3.log
python scripts/prof_eig.py --config 4 --reps 1 > gpurun_out/r02eigl/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "ks_pencil_eig/" --csv --log-file gpurun_out/r02eigl/launches_eig_c4.csv python scripts/prof_eig.py --config 4 --reps 1 > gpurun_out/r02eigl/ncu.log 2>&1
tail -3 gpurun_out/r02eigl/pytest_next3.log; tail -2 gpurun_out/r02eigl/plain.log; wc -l gpurun_out/r02eigl/launches_eig_c4.csv
