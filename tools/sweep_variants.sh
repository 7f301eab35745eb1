# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 300 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)"; }
run HCAMG_TRI_THREADS=512
run HCAMG_TRI_THREADS=384
run HCAMG_TRI_THREADS=256
run HCAMG_TRI_THREADS=384 HCAMG_TRI_PFMODE=0
run HCAMG_TRI_THREADS=384 HCAMG_TRI_DBG=1
