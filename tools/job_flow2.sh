for ns in 0 32 256; do echo "== HCAMG_FLOW_NS=$ns"; HCAMG_FLOW_NS=$ns python tools/trace_flow.py c1 | sed -n '1p;8,12p'; done
for ns in 0 32; do echo "== HCAMG_FLOW_NS=$ns blocks 148"; HCAMG_FLOW_BLOCKS=148 HCAMG_FLOW_NS=$ns python tools/trace_flow.py c1 | sed -n '1p;8,12p'; done
HCAMG_FLOW_NS=0 python tools/trace_flow.py c2 | sed -n '1p;8,12p;40,44p'
