mkdir -p gpurun_out/t2d
timeout 600 python -m pytest tests/test_gpu_amr.py -x -q 2>&1 | tail -2
timeout 900 python tools/amr_test2.py 600 3 0.01 design > gpurun_out/t2d/t2_tol01_design.json 2>&1; cut -c1-1200 gpurun_out/t2d/t2_tol01_design.json
timeout 600 python tools/test1_acceptance.py 400 3 0.002 design > gpurun_out/t2d/t1_design.json 2>&1; cut -c1-1500 gpurun_out/t2d/t1_design.json
