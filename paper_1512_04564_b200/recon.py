"""Device-side setup for one reconstruction: allocation + C-ABI calls only.

`Recon` owns the torch CUDA tensors (sinogram y, weights w, D_L, state x, g,
htilde, workspace) and the ct_geom handle, and calls the C-ABI in the order of
Algorithm 1: D_L once, then
oslalm_relaxed_solve for as many sub-iterations as asked (line 1 runs inside
the first call, k == 0).  No arithmetic of the method runs in Python.
"""
import math

import torch

from . import ctrecon as C


def _variant(solver):
    v = solver.get("variant", "proposed")
    if v not in ("proposed", "simple"):
        raise ValueError("solver variant must be 'proposed' (Algorithm 1) or 'simple' (Algorithm 2), got %r" % (v,))
    return C.SIMPLE if v == "simple" else C.PROPOSED


class Recon:
    def __init__(self, geom, reg, solver, y, w, x0, kappa=None, device=0, dist=None, stream=None,
                 fwd_segments=None):
        """geom/reg/solver: dicts as in synth/configs.py; y, w: (na, nt, ns);
        x0: (nz, ny, nx).  Arrays may be numpy/torch of any float dtype; they
        are copied to float32 device tensors.  fwd_segments: None = the library's
        automatic choice, else ct_geom_set_fwd_segments(nseg) (0 = off)."""
        self.dev = torch.device("cuda", device)
        self.geom = geom
        self.desc = C.geom_desc(geom)
        self.h = C.ct_geom_create(self.desc, device)
        if fwd_segments is not None:
            C.ct_geom_set_fwd_segments(self.h, fwd_segments)
        self.dist = dist
        self.stream = stream
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.y = torch.as_tensor(y).to(**f32).contiguous()
        self.w = torch.as_tensor(w).to(**f32).contiguous() if w is not None else None
        self.kappa = torch.as_tensor(kappa).to(**f32).contiguous() if kappa is not None else None
        self.x = torch.as_tensor(x0).to(**f32).contiguous().clone()
        self.g = torch.zeros_like(self.x)
        self.htilde = torch.zeros_like(self.x)
        self.reg = C.reg_desc(reg["potential"], reg["delta"], reg["betas"], reg["n_dirs"],
                              reg.get("curvature", "huber"), reg.get("q", 1.2))
        self.params = C.params(solver["M"], solver["alpha"],
                               C.RHO_FIXED if solver.get("rho_mode") == "fixed" else C.RHO_CONTINUATION,
                               solver.get("rho_fixed", 0.0),
                               C.INIT_FULL if solver.get("init_grad") == "full" else C.INIT_LAST_SUBSET,
                               solver.get("box_lo", 0.0), solver.get("box_hi", math.inf),
                               _variant(solver))
        nbytes = C.oslalm_workspace_size(self.h, self.params, dist)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        self.state = C.make_state(self.x, self.g, self.htilde, 0)
        self.dl = None

    def compute_DL(self):
        """D_L = diag(A'WA1) over all views (ct_sqs_diag), once per reconstruction."""
        self.dl = torch.empty_like(self.x)
        C.ct_sqs_diag(self.h, self.w, self.dl, self.ws, dist=self.dist, stream=self.stream)
        return self.dl

    def init_fbp(self):
        """x = FBP / FDK of y (ct_fbp; "an initial (FBP) image"): 2-D fan and
        axial cone scans with a 360-degree orbit.  Resets the solver state (k = 0)."""
        ws = torch.empty(self.y.numel() * 4, dtype=torch.uint8, device=self.dev)
        C.ct_fbp(self.h, self.y, self.x, ws, stream=self.stream)
        self.state.k = 0
        return self.x

    def set_DL(self, dl):
        self.dl = torch.as_tensor(dl).to(dtype=torch.float32, device=self.dev).contiguous()

    def run(self, n_subiters, x_ref=None, rms=None):
        if self.dl is None:
            self.compute_DL()
        C.oslalm_relaxed_solve(self.h, self.y, self.w, self.reg, self.kappa, self.dl, self.params, self.state,
                               n_subiters, self.ws, x_ref=x_ref, rms_per_iter=rms, dist=self.dist,
                               stream=self.stream)
        return self.x

    @property
    def k(self):
        return self.state.k

    def paper_h(self):
        h = torch.empty_like(self.x)
        C.oslalm_state_h(self.h, self.dl, self.state, h, stream=self.stream)
        return h

    def close(self):
        if self.h is not None:
            C.ct_geom_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostPipeline:
    """Host-resident data through the C-ABI with the copies hidden behind the
    solve: step i copies its (y, w) from pinned host memory into one of two
    device buffers on a copy stream while step i-1 computes on the other, runs
    `n_subiters` sub-iterations of `rec` on that data, snapshots x on the device
    and reads the snapshot back to pinned host memory on the copy stream.
    Every step moves its own inputs host->device and its result
    device->host; only the order is pipelined.  Allocation and CUDA stream /
    event plumbing only -- every arithmetic step is the C-ABI's."""

    def __init__(self, rec):
        self.rec = rec
        dev = rec.dev
        self.copy = torch.cuda.Stream(device=dev)
        self.comp = rec.stream if rec.stream is not None else torch.cuda.current_stream(dev)
        self.bufs = [(rec.y, rec.w), (torch.empty_like(rec.y), torch.empty_like(rec.w) if rec.w is not None else None)]
        self.snaps = [torch.empty_like(rec.x), torch.empty_like(rec.x)]
        self.copied = [torch.cuda.Event(), torch.cuda.Event()]
        self.used = [torch.cuda.Event(), torch.cuda.Event()]   # buffer i free again
        self.snapped = [torch.cuda.Event(), torch.cuda.Event()]
        self.read = [torch.cuda.Event(), torch.cuda.Event()]   # snapshot i read back
        for e in self.used + self.read:
            e.record(self.comp)
        self.sub_events = [None, None]
        self.i = 0

    def h2d_bytes(self, y_h, w_h):
        return y_h.numel() * y_h.element_size() + (w_h.numel() * w_h.element_size() if w_h is not None else 0)

    def enqueue_copy_in(self, y_h, w_h, by_subset=False):
        """Queue the host->device copy of the next step's inputs (buffer i % 2).
        by_subset: copy subset by subset (ct_sino_upload) in the order the next
        step visits them, with an event per subset, so that the step's first
        sub-iterations start before the whole sinogram has arrived (used for
        the first step, whose copy has no previous step to hide behind)."""
        b = self.i % 2
        rec = self.rec
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.used[b])
            if by_subset:
                M = rec.params.M
                na = rec.geom["na"]
                k = rec.state.k
                order = ([M - 1] if k == 0 else []) + [(k + q) % M for q in range(M)]
                evs = {}
                for m in order:
                    if m in evs:
                        continue
                    v = C.views(m, M, (na - m + M - 1) // M)
                    C.ct_sino_upload(rec.h, y_h, v, self.bufs[b][0], stream=self.copy)
                    if w_h is not None:
                        C.ct_sino_upload(rec.h, w_h, v, self.bufs[b][1], stream=self.copy)
                    e = torch.cuda.Event()
                    e.record(self.copy)
                    evs[m] = e
                self.sub_events[b] = evs
            else:
                self.bufs[b][0].copy_(y_h, non_blocking=True)
                if w_h is not None:
                    self.bufs[b][1].copy_(w_h, non_blocking=True)
                self.sub_events[b] = None
            self.copied[b].record(self.copy)

    def step(self, n_subiters, x_h, next_inputs=None):
        """Run step i on buffer i % 2 (its copy must have been enqueued), queue
        the copy of `next_inputs` = (y_h, w_h) for step i+1, read x back."""
        b = self.i % 2
        rec = self.rec
        rec.y, rec.w = self.bufs[b]
        evs = self.sub_events[b]
        if evs is None:
            self.comp.wait_event(self.copied[b])
        if next_inputs is not None:
            self.i += 1
            self.enqueue_copy_in(*next_inputs)
            self.i -= 1
        if evs is None:
            rec.run(n_subiters)
        else:
            # sub-iteration by sub-iteration, each after its subset's copy (k = 0 also reads subset M-1)
            M = rec.params.M
            if rec.dl is None or (rec.state.k == 0 and rec.params.init_grad == C.INIT_FULL):
                # D_L (all views) or the full-gradient line 1 reads every subset: the whole copy first
                self.comp.wait_event(self.copied[b])
            for _ in range(n_subiters):
                k = rec.state.k
                if k == 0:
                    self.comp.wait_event(evs[M - 1])
                self.comp.wait_event(evs[k % M])
                rec.run(1)
            self.comp.wait_event(self.copied[b])
            self.sub_events[b] = None
        self.used[b].record(self.comp)
        self.comp.wait_event(self.read[b])
        self.snaps[b].copy_(rec.x)
        self.snapped[b].record(self.comp)
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.snapped[b])
            x_h.copy_(self.snaps[b], non_blocking=True)
            self.read[b].record(self.copy)
        self.i += 1

    def finish(self):
        """Make the compute stream wait for every outstanding copy."""
        self.comp.wait_stream(self.copy)


class ZslabRecon:
    """Rank `rank` of a z-slab decomposition (oslalm_zslab_solve):
    holds this rank's planes of x, g, htilde, D_L and the full y, w.  Same
    run / compute_DL / x interface as Recon (allocation + C-ABI calls only).
    dist: a ct_dist communicator for world > 1 (one process per GPU)."""

    def __init__(self, geom, reg, solver, y, w, x0, rank=0, world=1, device=0, dist=None, stream=None):
        self.dev = torch.device("cuda", device)
        self.geom = geom
        self.h = C.ct_geom_create(C.geom_desc(geom), device)
        self.rank, self.world, self.dist, self.stream = rank, world, dist, stream
        self.z0, self.nz = C.ct_zslab_range(self.h, rank, world)
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.y = torch.as_tensor(y).to(**f32).contiguous()
        self.w = torch.as_tensor(w).to(**f32).contiguous()
        self.x = torch.as_tensor(x0).to(**f32)[self.z0:self.z0 + self.nz].contiguous().clone()
        self.g = torch.zeros_like(self.x)
        self.htilde = torch.zeros_like(self.x)
        self.dl = torch.empty_like(self.x)
        self.reg = C.reg_desc(reg["potential"], reg["delta"], reg["betas"], reg["n_dirs"],
                              reg.get("curvature", "huber"), reg.get("q", 1.2))
        self.params = C.params(solver["M"], solver["alpha"],
                               C.RHO_FIXED if solver.get("rho_mode") == "fixed" else C.RHO_CONTINUATION,
                               solver.get("rho_fixed", 0.0),
                               C.INIT_FULL if solver.get("init_grad") == "full" else C.INIT_LAST_SUBSET,
                               solver.get("box_lo", 0.0), solver.get("box_hi", math.inf),
                               _variant(solver))
        self.ws = torch.empty(C.oslalm_zslab_workspace_size(self.h, self.params, rank, world), dtype=torch.uint8,
                              device=self.dev)
        self.state = C.make_state(self.x, self.g, self.htilde, 0)
        self.have_dl = False

    def compute_DL(self):
        C.ct_sqs_diag_zslab(self.h, self.w, [self.dl], [self.ws], self.world, dist=self.dist, stream=self.stream)
        self.have_dl = True
        return self.dl

    def run(self, n_subiters):
        if not self.have_dl:
            self.compute_DL()
        C.oslalm_zslab_solve(self.h, self.y, self.w, self.reg, [self.dl], self.params, [self.state], n_subiters,
                             [self.ws], self.world, dist=self.dist, stream=self.stream)
        return self.x

    @property
    def k(self):
        return self.state.k

    def close(self):
        if self.h is not None:
            C.ct_geom_destroy(self.h)
            self.h = None
