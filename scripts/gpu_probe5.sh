timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python -c "
import ctypes; c=ctypes.CDLL('libcudart.so') if False else None
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)
"
OMCG_L2_PERSIST=0 python scripts/run_c2.py 7 2
OMCG_L2_PERSIST=1 python scripts/run_c2.py 7 2
