"""Run an oracle computation in a forked background process (test / bench
infrastructure, like the rest of oracle/).

The oracle is serial, so a full-length parity run takes minutes; forking it lets
the GPU work of the caller proceed meanwhile.  The child works on host numpy
arrays and the oracle's ctypes library only (it never touches CUDA), writes the
returned dict of arrays / scalars to an .npz and leaves with os._exit (no atexit
handlers of the parent, such as CUDA's, run in it)."""
from __future__ import annotations

import multiprocessing as mp
import os
import time
import traceback

import numpy as np


def _child(fn, path):
    try:
        out = fn()
        np.savez(path, **out)
        code = 0
    except BaseException:
        with open(path + ".err", "w") as f:
            f.write(traceback.format_exc())
        code = 1
    os._exit(code)


class Job:
    """fn() runs in a forked child and returns a dict of numpy arrays / scalars;
    result() waits for it and loads that dict (plus wall_s since the fork)."""

    def __init__(self, name, fn, tmpdir):
        self.name = name
        self.path = os.path.join(tmpdir, name + ".npz")
        self.t0 = time.time()
        self.proc = mp.get_context("fork").Process(target=_child, args=(fn, self.path), daemon=True)
        self.proc.start()
        self._res = None

    def done(self):
        return not self.proc.is_alive()

    def result(self, timeout=1800):
        if self._res is None:
            self.proc.join(timeout)
            if self.proc.is_alive():
                self.proc.kill()
                raise TimeoutError("oracle job %s still running after %d s" % (self.name, timeout))
            err = self.path + ".err"
            if os.path.exists(err):
                raise RuntimeError("oracle job %s failed:\n%s" % (self.name, open(err).read()))
            if self.proc.exitcode != 0 or not os.path.exists(self.path):
                raise RuntimeError("oracle job %s exited with %s" % (self.name, self.proc.exitcode))
            with np.load(self.path) as z:
                self._res = {k: z[k] for k in z.files}
            self._res["wall_s"] = time.time() - self.t0
        return self._res

    def kill(self):
        if self.proc.is_alive():
            self.proc.kill()
