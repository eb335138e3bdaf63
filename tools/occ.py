import ctypes, sys
sys.path.insert(0, ".")
import torch
from paper_2511_09741_b200 import tawpipe as T
L = T.lib()
cudart = ctypes.CDLL("libcudart.so.12") if False else None
print(torch.cuda.get_device_properties(0))
