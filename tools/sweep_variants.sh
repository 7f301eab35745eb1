# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)|rror"; }
run HCAMG_TRI_CRITW=140 HCAMG_TRI_TASKW=1536
run HCAMG_TRI_CRITW=140 HCAMG_TRI_TASKW=1024
run HCAMG_TRI_CRITW=140 HCAMG_TRI_TASKW=2048
run HCAMG_TRI_CRITW=160 HCAMG_TRI_TASKW=2048
run HCAMG_TRI_CRITW=150 HCAMG_TRI_TASKW=1536
