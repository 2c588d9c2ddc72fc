"""NEXT-1 measurement side: the per-bucket synchronisation timer of
PAPER.md:347-352 -- "an utility that measures time each bucket takes to synchronize ...
we measure gradients synchronization time for various combinations of compression
ratios per bucket, saving the communicated buckets sizes.  Then, we train a linear
regression model to learn the relation between the transmitted bucket sizes and the
gradient synchronization time" -- feeding `objectives.fit_bucket_time` and
`objectives.time_weights` (the weights `lgreco.weight_costs` multiplies into the size
table before `lgreco.solve`).

Device-timed: a CUDA event pair per bucket on the stream its synchronisation call runs
on; a step's gradient synchronisation time is the interval from the first bucket's
start to the last bucket's end (the last bucket's synchronisation is
the delay between steps).  Orchestration only -- the timed calls are the library's.
"""
import numpy as np
import torch


class BucketSyncTimer:
    def __init__(self, nbuckets=0):
        self.nb = int(nbuckets)  # grows with the largest bucket index seen
        self._steps = []  # [{bucket: [bytes, ev0, ev1]}]
        self._cur = None

    def begin_step(self):
        self._cur = {}

    def start(self, b, stream=None):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self._cur[b] = [0.0, ev, None]
        self.nb = max(self.nb, b + 1)

    def stop(self, b, sent_bytes, stream=None):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        self._cur[b][0] = float(sent_bytes)
        self._cur[b][2] = ev

    def end_step(self):
        if self._cur:
            self._steps.append(self._cur)
        self._cur = None

    def samples(self):
        """(sizes (S, nb) transmitted bytes per bucket, sync (S,) ms from the first bucket's
        start to the last bucket's end, per_bucket (S, nb) ms) of every recorded step
        (synchronises the device)."""
        torch.cuda.synchronize()
        sizes = np.zeros((len(self._steps), self.nb))
        per = np.zeros((len(self._steps), self.nb))
        sync = np.zeros(len(self._steps))
        for i, st in enumerate(self._steps):
            t0 = st[min(st)][1]
            for b, (by, e0, e1) in st.items():
                sizes[i, b] = by
                per[i, b] = e0.elapsed_time(e1)
                sync[i] = max(sync[i], t0.elapsed_time(e1))
        return sizes, sync, per


def r_squared(sizes, times, T, c):
    """Coefficient of determination of the fitted model times ~ sizes @ T + c."""
    pred = np.asarray(sizes) @ np.asarray(T) + c
    y = np.asarray(times, dtype=np.float64)
    ss = float(((y - y.mean()) ** 2).sum())
    return 1.0 - float(((y - pred) ** 2).sum()) / ss if ss > 0 else 1.0
