import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
import test_gpu_gather as t
world, H, p, delay, mode = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), sys.argv[4], sys.argv[5]
delay = None if delay == "none" else int(delay)
side = torch.cuda.Stream()
def sleep_same():  # sleep kernel on the current (default) stream, then event wait
    torch.cuda._sleep(20_000_000)
def host():
    time.sleep(0.01)
def host_long():
    time.sleep(0.5)
fn = {"host": host, "host_long": host_long, "sleep_default": sleep_same}[mode]
t0 = time.time()
try:
    t._virtual_ranks_fused(world, 4 * world, 197, H, p, iters=2, delay_rank=delay, delay_fn=fn)
    print("CASE", sys.argv[1:], "OK", round(time.time() - t0, 3))
except Exception as e:
    print("CASE", sys.argv[1:], "FAIL", round(time.time() - t0, 3), repr(e)[:120])
