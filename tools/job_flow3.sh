for g in 1 0; do for ns in 0 32; do echo "== gate $g ns $ns"; HCAMG_FLOW_GATE=$g HCAMG_FLOW_NS=$ns python tools/trace_flow.py c1 | sed -n '1p;/link latency/p'; HCAMG_FLOW_GATE=$g HCAMG_FLOW_NS=$ns python tools/profile_pieces.py c2 "" "opt:sweep=4" | grep leg; done; done
python tools/trace_flow.py c2 | sed -n '1,4p;30,34p;60,64p;90,100p'
