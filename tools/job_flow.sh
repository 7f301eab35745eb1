set -x
mkdir -p gpurun_out
timeout 600 python tools/profile_pieces.py c2 "" "opt:sweep=0,2,4" > gpurun_out/flow_pieces.log 2>&1
tail -30 gpurun_out/flow_pieces.log
timeout 600 python tools/profile_pieces.py c1 "" "opt:sweep=0,1,2,4" > gpurun_out/flow_pieces_c1.log 2>&1
tail -30 gpurun_out/flow_pieces_c1.log
