"""e2e breakdown of pb_batch_run on the 4096 batch (pack + H2D + walk + D2H),
repeated to exercise buffer reuse across runs."""
import sys, time; sys.path.insert(0, '.')
import paper_2312_06902_b200 as pb
from paper_2312_06902_b200 import g9
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
b = pb.FrontierBatch()
t = time.time()
for i in range(4096): b.add_g9(g9.batch_params(i))
print(f"add (validate+derive) {time.time()-t:.2f}s", flush=True)
for rep in range(reps):
    t = time.time(); b.run(0); wall = time.time() - t
    st = b.stats()
    print(f"run {rep} wall {wall:.2f}s kernel {st.kernel_ms/1e3:.2f}s h2d {st.h2d_ms/1e3:.2f}s ({st.h2d_bytes/1e9:.2f} GB) "
          f"d2h {st.d2h_ms/1e3:.2f}s ({st.d2h_bytes/1e9:.2f} GB)", flush=True)
