cd $GRAFT_REPO_ROOT
for FL in "" "-DTOMESH_EXP_ONE_CTA"; do
  sed -i "s|^NVCC_FLAGS = \[.*|NVCC_FLAGS = [\"-DEXPDUMMY\", $(for f in $FL; do printf '"%s", ' $f; done)|" paper_1009_4975_b200/build.py
  python -c "from paper_1009_4975_b200 import build; build.build(force=True)"
  echo "FLAGS: $FL"; python tools/microbench.py c5 | cut -c1-200
done
