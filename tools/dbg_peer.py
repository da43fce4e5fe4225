import os, sys, socket
sys.path.insert(0, os.getcwd())
import numpy as np
import torch.multiprocessing as mp

def worker(rank, world, port, q):
    import torch, torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2112_01579_b200 as P
    from paper_2112_01579_b200.sharding import PeerFrameRenderer
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=16, seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    print("rank", rank, src.device_model.info(), flush=True)
    pad = torch.empty(40000, dtype=torch.float32, device="cuda")
    r = PeerFrameRenderer(src)
    cams = P.fibonacci_cameras(8, 203, 157)
    got = []
    for v in (3, 4, 5):
        out = r.render(cams[v], P.RenderSettings(stepsize=1 / 128), count=True)
        if rank == 0:
            got.append((out.cpu().numpy(), r.last_eval_count))
    if rank == 0: q.put(got)
    dist.barrier(); r.close(); dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    import paper_2112_01579_b200 as P
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    [p.start() for p in ps]
    got = q.get(timeout=300); [p.join() for p in ps]
    m = P.model_init(P.ModelConfig(layers=4, hidden=32, grid_resolution=16, seed=0))
    src = P.ModelSource(m, P.TF_PRESETS["warm"])
    print("main", src.device_model.info())
    cams = P.fibonacci_cameras(8, 203, 157)
    for (frame, count), v in zip(got, (3, 4, 5)):
        img = P.render_image(src, cams[v], P.RenderSettings(stepsize=1 / 128)).data
        d = np.abs(frame - img)
        bad = np.argwhere(d.max(-1) > 0)
        print(v, "maxdiff", d.max(), "npix", len(bad), "count", count, src.last_eval_count, bad[:5].tolist())
        if len(bad):
            tiles = {(int(y)//8, int(x)//8) for y, x in bad}
            print("  tiles", sorted(tiles)[:10], len(tiles), "zero pixels in frame", int((frame.max(-1) == 0).sum()), int((img.max(-1)==0).sum()))
