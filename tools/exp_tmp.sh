cd $GRAFT_REPO_ROOT
sed -i 's|^NVCC_FLAGS = \[.*|NVCC_FLAGS = ["-DTOMESH_EXP_FIXED_SCALARS", "-DTOMESH_EXP_NO_ELEMENT",|' paper_1009_4975_b200/build.py
python -c "from paper_1009_4975_b200 import build; build.build(force=True)"
python tools/prof_run.py c5 3 && ncu --set full --import-source on --clock-control none -k regex:k_apply_s3 -s 2 -c 1 -o gpurun_out/noelem python tools/prof_run.py c5 3 > /dev/null 2>&1; ls gpurun_out
