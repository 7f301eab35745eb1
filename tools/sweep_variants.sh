# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)|rror"; }
run HCAMG_TRI_KERNEL=2
run HCAMG_TRI_KERNEL=2 HCAMG_TRI_CRITW=120
run HCAMG_TRI_KERNEL=2 HCAMG_TRI_TASKW=2048
