# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)|rror"; }
run HCAMG_TRI_SLOTS=2
run HCAMG_TRI_SLOTS=2 HCAMG_TRI_TASKW=1536
run HCAMG_TRI_SLOTS=2 HCAMG_TRI_TASKW=6144
run HCAMG_TRI_SLOTS=2 HCAMG_TRI_CRITW=120
run HCAMG_TRI_SLOTS=2 HCAMG_TRI_CRITW=160
run HCAMG_TRI_SLOTS=2 HCAMG_TRI_L2PF=1
run HCAMG_TRI_SLOTS=2 HCAMG_TRI_L2PF=0
