import sys, numpy as np, torch, ctypes as C
sys.path.insert(0, ".")
import oracle
from paper_1709_08990_b200 import gen
from paper_1709_08990_b200._native import lib
from paper_1709_08990_b200.device import DeviceCodec, ENCODE_SEG_DTYPE, segments_to_tensor
dev = DeviceCodec(0)
lib.bcgpu_debug_set_flags.argtypes = [C.c_void_p, C.c_uint32]
nl = int(sys.argv[1]); flags = int(sys.argv[2], 0)
lb = gen.posting_lists(nl, 4, cap_total=nl * 1024)
lists = [lb.values[int(lb.offsets[i]):int(lb.offsets[i + 1])] for i in range(nl)]
caps = np.array([(v.size + 3) // 4 + 4 * v.size for v in lists], np.uint64)
eoff = np.concatenate([[0], np.cumsum(caps)])
es = np.zeros(nl, ENCODE_SEG_DTYPE)
es["src_offset"], es["dst_capacity"], es["dst_offset"] = lb.offsets[:-1], caps, eoff[:-1]
es["n"], es["prev"] = lb.lengths, 0
d_vals = torch.from_numpy(lb.values.view(np.int32).copy()).cuda()
d_enc = torch.zeros(int(eoff[-1]) + 16, dtype=torch.uint8, device="cuda")
d_lens = torch.zeros(nl, dtype=torch.int64, device="cuda")
lib.bcgpu_debug_set_flags(dev._ctx, flags)
dev.encode_batch(segments_to_tensor(es, "cuda"), nl, d_vals, d_enc, d_lens, delta=True, max_seg_n=int(lb.lengths.max()))
dev.check()
h = d_enc.cpu().numpy(); lens = d_lens.cpu().numpy()
nbad = 0
for i, v in enumerate(lists):
    e = oracle.encode(v, delta=True, prev=0)
    got = h[int(eoff[i]):int(eoff[i]) + len(e)].tobytes()
    if got != e or lens[i] != len(e):
        nbad += 1
        if nbad <= 3:
            a = np.frombuffer(got, np.uint8); b = np.frombuffer(e, np.uint8)
            d = np.nonzero(a != b)[0]
            print(f"seg {i} n={v.size} ngroups={(v.size+3)//4} len={len(e)} got_len={lens[i]} ndiff={d.size} first={d[:8]} dst={int(eoff[i])} src={int(lb.offsets[i])}")
print("bad segments", nbad, "of", nl)
