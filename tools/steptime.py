import sys, time, torch
sys.path.insert(0, '/root/repo')
import bench, paper_2111_09562_b200 as pb
torch.cuda.set_device(0)
ts, ebs, info, _ = bench.build_workload("alexnet256", "cuda")
ps = [pb.CodecParams(eb=e) for e in ebs]
outs = [torch.empty_like(t) for t in ts]
for it in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    comp = pb.compress_batch(ts, ps)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    for (c, r), o in zip(comp, outs): pb.decompress_device(c, out=o, check=False)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"step {it}: compress {1e3*(t1-t0):.2f} ms  decompress {1e3*(t2-t1):.2f} ms  mem {torch.cuda.memory_allocated()/1e9:.2f} GB reserved {torch.cuda.memory_reserved()/1e9:.2f}")
