"""Print the per-tile phase breakdown of a recurrence trace [T][16] (see rec_tc*.cu SL_TRACE)."""
import torch


def report(buf, T, name):
    t = buf.view(T, 16).cpu().double()
    rel = (t - t[1, 0].item()) / 1000.0
    med = lambda x: x[2:-1].median().item()
    print(f"{name}: period {med(rel[2:,0]-rel[1:-1,0]):.2f} us | tile0: wait->first {med(rel[:,1]-rel[:,0]):.2f} "
          f"stream {med(rel[:,2]-rel[:,1]):.2f} mma->pub {med(rel[:,6]-rel[:,2]):.2f} | tile1: wait->first "
          f"{med(rel[:,4]-rel[:,3]):.2f} stream {med(rel[:,5]-rel[:,4]):.2f} mma->pub {med(rel[:,7]-rel[:,5]):.2f} | "
          f"t1 start after t0 pub {med(rel[:,3]-rel[:,6]):.2f}")
    if t[2:-1, 8].min() > 0:
        print(f"   epi tile0: loop-start->tfull {med(rel[:,8]-rel[:,12]):.2f} (last MMA issue->tfull "
              f"{med(rel[:,8]-rel[:,2]):.2f}) sends {med(rel[:,9]-rel[:,8]):.2f} "
              f"recv-wait {med(rel[:,10]-rel[:,9]):.2f} math+stores {med(rel[:,11]-rel[:,10]):.2f} "
              f"sync+pub {med(rel[:,6]-rel[:,11]):.2f}")
    if t[2:-1, 13].min() > 0 and t[2:-1, 14].min() > 0:
        print(f"   math detail: recv-read {med(rel[:,13]-rel[:,10]):.2f} compute {med(rel[:,14]-rel[:,13]):.2f} "
              f"ring-store {med(rel[:,11]-rel[:,14]):.2f}")
