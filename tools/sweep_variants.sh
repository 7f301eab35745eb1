# time the dense-regime sweeps (level-0 restriction / prolongation) under kernel knobs
run() { echo "== $*"; env "$@" timeout 120 python tools/profile_pieces.py c2 2>&1 | grep -E "L0 (prolong)|rror"; }
run HCAMG_TRI_TMEM=0
run HCAMG_TRI_TMEM=1
run HCAMG_TRI_TMEM=1 HCAMG_TRI_SLOTS=3
