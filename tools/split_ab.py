import sys, os
sys.path.insert(0, '/root/repo/tools'); sys.path.insert(0, '/root/repo')
import attn_check as A
libs = [("sw2", "paper_2603_05353_b200/_build/libifkv.so"), ("sw1", "_ab/sw1/libifkv.so"), ("sw3", "_ab/sw3/libifkv.so"), ("sw4", "_ab/sw4/libifkv.so")]
for k in (1639, 2458, 3277, 4916):
    for rep in range(3):
        for name, lib in libs:
            E = A.use(lib, 10)
            ms, tf, out = A.time_c2(E, k=k)
            print(f"k={k} rep{rep} {name}: {ms:.3f} ms {tf:.0f} TF/s", flush=True)
