cd paper_2402_09222_b200/csrc && touch kernels.cu && make -s KFLAGS=-DOMCG_MOVE_CYCLES 2>&1 | grep -E "error" ; cd ../..
OMCG_MOVE_CYCLES=1 python scripts/gap.py 2>&1 | tail -12
