# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)|rror"; }
run HCAMG_TRI_BAR=0
run HCAMG_TRI_BAR=1
run HCAMG_TRI_BAR=2
run HCAMG_TRI_BAR=0 HCAMG_TRI_L2PF=0
run HCAMG_TRI_BAR=0 HCAMG_TRI_L2PF=2
