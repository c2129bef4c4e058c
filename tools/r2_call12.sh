T="timeout 300 python -m pytest tests/test_gpu_edge_cases.py -x -q -k k_equals_prompt"
echo "default"; $T 2>&1 | tail -1
echo "pdl0"; CLO_PDL=0 $T 2>&1 | tail -1
echo "noov"; CLO_GATHER_OVERLAP=0 $T 2>&1 | tail -1
echo "nt"; CLO_LIB=paper_2511_14510_b200/libclo_nt.so $T 2>&1 | tail -1
echo "lsu"; CLO_GATHER=lsu $T 2>&1 | tail -1
