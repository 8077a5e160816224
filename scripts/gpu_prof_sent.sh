cat > /tmp/sent.py <<'PY'
import sys; sys.path.insert(0, "/root/repo")
import torch, paper_2605_01708_b200 as sz
from paper_2605_01708_b200.engine import DeviceCodec, synth_kv
fmt = sz.ElementFormat.BF16
bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
n = 1 << 28
w = synth_kv(n, fmt, 3, bw, esc, 0.0016)
m = sz.CodebookMode.TOP15_SENTINEL
book = sz.ExponentCodebook(fmt, tuple(e for e, _ in bw)[:15], 4, m)
cfg = sz.CodecConfig(fmt, 4, m, 1024, codebook=book)
eng = DeviceCodec(cfg, book, n); eng.ensure_capacity(w)
for _ in range(3): eng.decode()
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --clock-control none -k regex:'decode_persistent|marks_kernel|offsets' -s 3 -c 3 -o gpurun_out/prof_sent python /tmp/sent.py > /dev/null 2>&1
ls gpurun_out/prof_sent*
