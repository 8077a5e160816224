import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2605_01708_b200 as m
from paper_2605_01708_b200 import _native as N, peer
from paper_2605_01708_b200.engine import synth_kv
lib = N.load_library()
flag = torch.zeros(4, dtype=torch.int64, device="cuda")
to = torch.zeros(1, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.time()
N.check(lib.sz_peer_wait(N.ptr(flag), 1, int(3e9), N.ptr(to), s2.cuda_stream), "w")
N.check(lib.sz_peer_signal(N.ptr(flag), 1, s1.cuda_stream), "s")
torch.cuda.synchronize()
print("exp1 signal-only: %.3fs timed_out=%d" % (time.time() - t, to.item()), flush=True)
# exp2: wait on s2, heavy encode on s1 then signal
fmt = m.ElementFormat.BF16
bw, esc = tuple((0x70 + i, 0.72 ** i) for i in range(16)), tuple(range(0x10, 0x18))
words = synth_kv(1 << 24, fmt, 1, bw, esc, 0.0016)
book = m.ExponentCodebook(fmt, tuple(e for e, _ in bw), 4, m.CodebookMode.TOPK_EXPLICIT)
cfg = m.CodecConfig(fmt, codebook=book)
from paper_2605_01708_b200.engine import DeviceCodec
eng = DeviceCodec(cfg, book, 1 << 24)
to.zero_(); flag.zero_(); torch.cuda.synchronize()
t = time.time()
N.check(lib.sz_peer_wait(N.ptr(flag) + 8, 1, int(3e9), N.ptr(to), s2.cuda_stream), "w")
with torch.cuda.stream(s1):
    eng.encode(words, stream=s1)
N.check(lib.sz_peer_signal(N.ptr(flag) + 8, 1, s1.cuda_stream), "s")
torch.cuda.synchronize()
print("exp2 encode-then-signal: %.3fs timed_out=%d" % (time.time() - t, to.item()), flush=True)
# exp3: decode on s2 concurrently with a wait on s1
to.zero_(); flag.zero_(); eng.encode(words); torch.cuda.synchronize()
t = time.time()
N.check(lib.sz_peer_wait(N.ptr(flag) + 16, 1, int(3e9), N.ptr(to), s1.cuda_stream), "w")
eng.decode(stream=s2)
N.check(lib.sz_peer_signal(N.ptr(flag) + 16, 1, s2.cuda_stream), "s")
torch.cuda.synchronize()
print("exp3 decode-then-signal: %.3fs timed_out=%d" % (time.time() - t, to.item()), flush=True)
# exp4: loopback link, 1 piece, 3 s timeout
snd, rcv = peer.connect_pair("send", 0, 1 << 20, cfg, book, slots=2, loopback=True, timeout_s=3)
w = words[: 1 << 20].clone()
out = torch.zeros_like(w)
torch.cuda.synchronize()
t = time.time()
rcv.recv(out, stream=s2)
snd.send(w, stream=s1)
torch.cuda.synchronize()
print("exp4 loopback 1 piece: %.3fs snd_to=%d rcv_to=%d equal=%s ready=%s free=%s" % (
    time.time() - t, snd.timed_out.item(), rcv.timed_out.item(), torch.equal(out, w),
    rcv.s.ready.tolist(), snd.free.tolist()), flush=True)
