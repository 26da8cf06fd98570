import itertools, collections
S, PPW = 6, 5
PPT = 4*PPW
def row0(pt): return (pt//PPW)*32 + (pt%PPW)*S
def wf128(addrs_bytes):  # 32 lanes, 16-byte accesses, 4 phases of 8
    tot=0
    for ph in range(4):
        a=addrs_bytes[ph*8:(ph+1)*8]
        c=collections.Counter((x//16)%8 for x in set(a))
        tot+=max(c.values())
    return tot
def wf32(addrs_bytes):
    c=collections.Counter((x//4)%32 for x in set(addrs_bytes))
    return max(c.values())
def fwd_quad(QS, mapping, ITEMS=80):
    # per stream s: vload 16B at (kq*QS + row0(pt)*4 + 4s)*4 bytes
    total=0; ideal=0
    for w0 in range(0, 128, 32):
        items=[w0+l for l in range(32)]
        items=[i for i in items if i < ITEMS]
        if not items: continue
        items += [items[-1]]*(32-len(items))
        for s in range(S):
            addrs=[(kq*QS + row0(pt)*4 + 4*s)*4 for pt,kq in (mapping(i) for i in items)]
            total+=wf128(addrs); ideal+=4
    return total, ideal
orig=lambda i: (i % PPT, i // PPT)
def alt(i):
    a,r=divmod(i,16); b,r=divmod(r,8); c,d=divmod(r,2)
    return (c + 4*a, d + 2*b)
def alt2(i):
    # 8 lanes: (kq 0..3, 2 points apart); interleave
    kq = i % 4; pt = i // 4
    return (pt, kq)
for QS in (512,516,520,528):
    for name,m in (("orig",orig),("alt",alt),("alt2",alt2)):
        print(QS, name, fwd_quad(QS,m))
# St gather: item=(rq,k16): src=(k16>>2)*QS + 16*rq + (k16&3) + 4*rr  (floats), rr=0..3 scalar loads
def st_gather(QS):
    tot=0
    for it in range(4):
        for w0 in range(0,128,32):
            items=[it*128+w0+l for l in range(32)]
            for rr in range(4):
                addrs=[((k16>>2)*QS + 16*(item>>4) + (k16&3) + 4*rr)*4 for item in items for k16 in [item&15]]
                tot+=wf32(addrs)
    return tot, 4*4*4
for QS in (512,516,520,528):
    print("stgather", QS, st_gather(QS))
