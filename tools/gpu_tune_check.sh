cp ab/lib_${TUNE_LIB:-tune}.so paper_1009_4975_b200/libtomesh.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amr.py -x -q 2>&1 | tail -1
python - <<'PY'
import paper_1009_4975_b200 as pb
from inputs import config
for args in [("c4", {}), ("c4", dict(base=(8,4,4), L=3, n_gauss=30)), ("c4", dict(base=(8,4,4), L=2, n_gauss=30))]:
    p = config(args[0], **args[1]); hm = pb.prepare(p)
    m = pb.Mesh(hm, E0=p.E0, Emin=p.Emin, nu=p.nu, rmin=p.rmin)
    print(hm.n_el, m.info()["matvec_variant"])
PY
bash tools/gen_ab_multi.sh tuneab${TUNE_LIB:-} tune ${TUNE_LIB:-tune}
