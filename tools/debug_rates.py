import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_15949_b200.network import LaudNetwork, random_images
net = LaudNetwork("resnet101", "spatial", "4-2-2-1", 0.5)
img = random_images(4)
rec = []
net.forward(img, record=rec); torch.cuda.synchronize()
for slot, c, cnt in rec[:3]:
    print(slot.stage, slot.index, c[:20].tolist(), cnt.tolist(), slot.db.masker_bias)
b = net.calibrate(img); print("biases", b[:5])
rec = []
net.forward(img, record=rec); torch.cuda.synchronize()
for slot, c, cnt in rec[:3]:
    print(slot.stage, slot.index, c[:20].tolist(), cnt.tolist(), slot.db.masker_bias)
print(net.rate_stats(img)[:4])
