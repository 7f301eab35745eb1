# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)|rror|sweep"; }
run HCAMG_SETUP_TIMING=1
run HCAMG_TRI_SLOTS=4
run HCAMG_TRI_SLOTS=2
run HCAMG_TRI_KERNEL=0
