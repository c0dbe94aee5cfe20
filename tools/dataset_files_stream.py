"""Dataset files at scale (headerless 8 MiB .bin files of 512 SwissSPAD2 frames;
SURVEY §8(f) f4): write F files of distinct synthetic frames to a scratch directory, then time
dataset.scan_dataset + dataset.correlate_files through one kind::mxf4 context (256^2 x 256^2,
CPI_KEEP_COUNTS, 65,536-frame batches spanning files: cpi_read_bin into two pinned buffers while
the GPU correlates the previous batch) and cpi_finalize.  Checks sum_pq S_ab = sum_i n_A(i) n_B(i)
exactly.  Prints one JSON line.  Env: CPI_DS_FILES (default 256 = 131,072 frames), CPI_DS_DIR."""
import json, os, shutil, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_2407_20692_b200 import Context, dataset

F = int(os.environ.get("CPI_DS_FILES", 256))
root = os.environ.get("CPI_DS_DIR") or tempfile.mkdtemp(prefix="cpi_ds_")
popc = np.array([bin(b).count("1") for b in range(256)], dtype=np.int64)
t0 = time.time()
closed = 0
for f in range(F):
    fr = synth.bernoulli_frames(512, 0.05, seed=synth.SEED_ARMS, frame0=512 * f)
    na = popc[fr[:, :, :32]].sum(axis=(1, 2))
    nb = popc[fr[:, :, 32:]].sum(axis=(1, 2))
    closed += int((na * nb).sum())
    with open(os.path.join(root, f"frames_{f:05d}.bin"), "wb") as fh:
        fh.write(fr.tobytes())
write_s = time.time() - t0
ctx = Context(synth.ROI_FULL_A, synth.ROI_FULL_B, 65536, variant="fp4", keep_counts=True)
t1 = time.time()
m = dataset.scan_dataset(root)
scan_s = time.time() - t1
# warm-up on the first batch, then the timed pass over every file
dataset.correlate_files(ctx, dataset.Manifest(m.file_paths[:128], m.frames_per_file))
torch.cuda.synchronize()
ctx.reset()
t2 = time.time()
n = dataset.correlate_files(ctx, m)
g = ctx.new_gamma()
n_tot = ctx.finalize(g)
torch.cuda.synchronize()
run_s = time.time() - t2
s_ab, _, _ = ctx.counts_views()
total = sum(int(s_ab[r:r + 4096].sum(dtype=torch.int64).item()) for r in range(0, s_ab.shape[0], 4096))
shutil.rmtree(root, ignore_errors=True)
print(json.dumps({"files": F, "frames": n, "n_tot": n_tot, "bytes": F * 8388608, "write_s": write_s, "scan_s": scan_s,
                  "stream_and_finalize_s": run_s, "frames_per_s": n / run_s,
                  "file_gbs": F * 8388608 / run_s / 1e9, "sum_s_ab": total, "closed_form": closed,
                  "exact": total == closed}))
