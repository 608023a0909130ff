"""Per-layer CPU/GPU expert placement (drop-in for reference assignment.py).

``greedy_assign`` runs the single-CTA greedy kernel (``dali_greedy``):
cost evaluation, the stable |t_gpu - t_cpu| ordering and Algorithm 1 all
happen on device.  The reference's comparison solvers -- beam search,
branch-and-bound ``optimal_assign`` and the static threshold -- run in the
same single-CTA kernel family (``dali_assign``).  ``validate`` /
``makespan`` are host-side constraint checks (assignment.py:126-169);
``all_cpu_assign`` / ``all_gpu_assign`` are the trivial baselines.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .cost_model import CostModel
from .errors import AssignmentError, ConstraintViolation

EXACT_SOLVER_LIMIT = 24          # assignment.py:23


@dataclass
class Assignment:
    """C[i] = 1 for CPU, G[i] = 1 for GPU (assignment.py:26-50)."""

    C: np.ndarray
    G: np.ndarray

    def __post_init__(self):
        self.C = np.asarray(self.C, dtype=np.int8)
        self.G = np.asarray(self.G, dtype=np.int8)
        if self.C.shape != self.G.shape:
            raise AssignmentError("C and G must have the same length")

    @property
    def cpu_indices(self) -> np.ndarray:
        return np.flatnonzero(self.C)

    @property
    def gpu_indices(self) -> np.ndarray:
        return np.flatnonzero(self.G)

    def __eq__(self, other) -> bool:
        return (isinstance(other, Assignment) and np.array_equal(self.C, other.C)
                and np.array_equal(self.G, other.G))


@dataclass
class AssignmentInstance:
    """One layer's placement problem (assignment.py:53-123)."""

    workloads: np.ndarray
    resident: np.ndarray
    cost_model: CostModel | None = None
    gpu_capacity: int | None = None
    _cpu_times: np.ndarray | None = field(default=None, repr=False)
    _gpu_times: np.ndarray | None = field(default=None, repr=False)
    _order: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        self.workloads = np.asarray(self.workloads, dtype=np.int64)
        self.resident = np.asarray(self.resident, dtype=bool)
        if self.workloads.shape != self.resident.shape:
            raise AssignmentError(f"workloads ({self.workloads.shape}) and resident flags "
                                  f"({self.resident.shape}) must share length")
        if (self.workloads < 0).any():
            raise AssignmentError("workloads must be nonnegative")
        if self.gpu_capacity is not None and self.gpu_capacity < 0:
            raise AssignmentError("gpu_capacity must be >= 0")
        if self._cpu_times is None:
            if self.cost_model is None:
                raise AssignmentError("either a cost model or explicit times required")
            # times are produced by the same device evaluation greedy uses
            _, _, order, times = _run_greedy(self, want_times=True)
            n = self.n_experts
            self._cpu_times, self._gpu_times = times[:n], times[n:]
            self._order = order

    @classmethod
    def from_times(cls, cpu_times, gpu_times, workloads=None, resident=None,
                   gpu_capacity=None) -> "AssignmentInstance":
        cpu_times = np.asarray(cpu_times, dtype=np.float64)
        gpu_times = np.asarray(gpu_times, dtype=np.float64)
        if cpu_times.shape != gpu_times.shape:
            raise AssignmentError("time vectors must share length")
        n = len(cpu_times)
        if workloads is None:
            workloads = ((cpu_times > 0) | (gpu_times > 0)).astype(np.int64)
        if resident is None:
            resident = np.zeros(n, dtype=bool)
        inst = cls.__new__(cls)
        inst.workloads = np.asarray(workloads, dtype=np.int64)
        inst.resident = np.asarray(resident, dtype=bool)
        inst.cost_model = None
        inst.gpu_capacity = gpu_capacity
        inst._cpu_times = cpu_times
        inst._gpu_times = gpu_times
        inst._order = None
        return inst

    @property
    def n_experts(self) -> int:
        return len(self.workloads)

    @property
    def cpu_times(self) -> np.ndarray:
        return self._cpu_times

    @property
    def gpu_times(self) -> np.ndarray:
        return self._gpu_times

    @property
    def activated(self) -> np.ndarray:
        return np.flatnonzero(self.workloads > 0)

    def sorted_order(self) -> np.ndarray:
        """Activated experts by descending |t_gpu - t_cpu|, ties to lower index
        (computed by the greedy kernel's ranking pass)."""
        if self._order is None:
            self._order = _run_greedy(self)[2]
        return self._order


def _run_greedy(inst: AssignmentInstance, want_times: bool = False):
    n = inst.n_experts
    if n > _lib.MAX_EXPERTS:
        raise AssignmentError(f"at most {_lib.MAX_EXPERTS} experts supported, got {n}")
    if n == 0:
        z = np.zeros(0, np.int8)
        return z, z, np.zeros(0, np.int64), np.zeros(0)
    w = _dev.to_dev(inst.workloads, torch.int64)
    r = _dev.to_dev(inst.resident.astype(np.uint8), torch.uint8)
    use_times = getattr(inst, "_cpu_times", None) is not None and not want_times
    ct = _dev.to_dev(inst._cpu_times, torch.float64) if use_times else None
    gt = _dev.to_dev(inst._gpu_times, torch.float64) if use_times else None
    Cd = _dev.empty((n,), torch.int8)
    Gd = _dev.empty((n,), torch.int8)
    od = _dev.empty((n,), torch.int32)
    td = _dev.empty((2 * n,), torch.float64) if want_times else None
    cm = inst.cost_model.to_c() if inst.cost_model is not None else None
    cap = -1 if inst.gpu_capacity is None else int(inst.gpu_capacity)
    _lib.call("dali_greedy", w.data_ptr(), r.data_ptr(), n, cap,
              C.addressof(cm) if cm is not None else None, _dev.ptr(ct), _dev.ptr(gt),
              Cd.data_ptr(), Gd.data_ptr(), od.data_ptr(), _dev.ptr(td), _dev.stream_ptr())
    order = od.cpu().numpy()
    order = order[order >= 0].astype(np.int64)
    return (Cd.cpu().numpy(), Gd.cpu().numpy(), order,
            td.cpu().numpy() if td is not None else None)


def greedy_assign(instance: AssignmentInstance) -> Assignment:
    """Completion-time greedy placement on device (assignment.py:172-199)."""
    C_, G_, order, _ = _run_greedy(instance)
    if instance._order is None:
        instance._order = order
    return Assignment(C=C_, G=G_)


def validate(instance: AssignmentInstance, assignment: Assignment) -> list[str]:
    """Every violated placement constraint (assignment.py:126-155)."""
    out = []
    C_, G_ = assignment.C, assignment.G
    if len(C_) != instance.n_experts:
        return [f"length mismatch: assignment has {len(C_)} experts, "
                f"instance has {instance.n_experts}"]
    for i in np.flatnonzero((C_ + G_) > 1):
        out.append(f"mutual exclusion violated at expert {i} (C=G=1)")
    for i in np.flatnonzero((C_ < 0) | (C_ > 1) | (G_ < 0) | (G_ > 1)):
        out.append(f"non-binary entry at expert {i}")
    n_assigned = int((C_ + G_).sum())
    n_act = int((instance.workloads > 0).sum())
    if n_assigned != n_act:
        out.append(f"activation count violated: {n_assigned} assigned vs {n_act} activated")
    for i in np.flatnonzero((instance.workloads > 0) & ((C_ + G_) == 0)):
        out.append(f"activation constraint violated: activated expert {i} unassigned")
    for i in np.flatnonzero((instance.workloads == 0) & ((C_ + G_) > 0)):
        out.append(f"unactivated expert {i} assigned")
    if instance.gpu_capacity is not None:
        new = int((G_.astype(bool) & ~instance.resident).sum())
        if new > instance.gpu_capacity:
            out.append(f"GPU capacity violated: {new} newly transferred experts > capacity "
                       f"{instance.gpu_capacity}")
    return out


def makespan(instance: AssignmentInstance, assignment: Assignment):
    """(T_cpu, T_gpu, T_layer) of a valid assignment (assignment.py:158-169)."""
    v = validate(instance, assignment)
    if v:
        raise ConstraintViolation(v)
    t_cpu = float(instance.cpu_times @ assignment.C)
    t_gpu = float(instance.gpu_times @ assignment.G)
    return t_cpu, t_gpu, max(t_cpu, t_gpu)


def all_cpu_assign(instance: AssignmentInstance) -> Assignment:
    n = instance.n_experts
    C_ = np.zeros(n, np.int8)
    C_[instance.activated] = 1
    return Assignment(C=C_, G=np.zeros(n, np.int8))


def all_gpu_assign(instance: AssignmentInstance) -> Assignment:
    n = instance.n_experts
    C_ = np.zeros(n, np.int8)
    G_ = np.zeros(n, np.int8)
    slots = instance.gpu_capacity
    for idx in instance.activated:
        if slots is None or slots > 0 or bool(instance.resident[idx]):
            G_[idx] = 1
            if slots is not None and not instance.resident[idx]:
                slots -= 1
        else:
            C_[idx] = 1
    return Assignment(C=C_, G=G_)


def _run_policy(inst: AssignmentInstance, policy: int, beam_width: int = 2,
                limit: int = EXACT_SOLVER_LIMIT, threshold: float | None = None):
    """Launch ``dali_assign`` for one instance -> (C, G, nodes)."""
    n = inst.n_experts
    if n > _lib.MAX_EXPERTS:
        raise AssignmentError(f"at most {_lib.MAX_EXPERTS} experts supported, got {n}")
    if n == 0:
        z = np.zeros(0, np.int8)
        return z, z, 0
    w = _dev.to_dev(inst.workloads, torch.int64)
    r = _dev.to_dev(inst.resident.astype(np.uint8), torch.uint8)
    use_times = getattr(inst, "_cpu_times", None) is not None
    ct = _dev.to_dev(inst._cpu_times, torch.float64) if use_times else None
    gt = _dev.to_dev(inst._gpu_times, torch.float64) if use_times else None
    Cd = _dev.empty((n,), torch.int8)
    Gd = _dev.empty((n,), torch.int8)
    nd = _dev.zeros((1,), torch.int64)
    cm = inst.cost_model.to_c() if inst.cost_model is not None else None
    cap = -1 if inst.gpu_capacity is None else int(inst.gpu_capacity)
    _lib.call("dali_assign", policy, w.data_ptr(), r.data_ptr(), n, cap,
              C.addressof(cm) if cm is not None else None, _dev.ptr(ct), _dev.ptr(gt),
              int(beam_width), int(limit), int(threshold is not None),
              float(threshold) if threshold is not None else 0.0, Cd.data_ptr(), Gd.data_ptr(),
              nd.data_ptr(), _dev.stream_ptr())
    return Cd.cpu().numpy(), Gd.cpu().numpy(), int(nd.cpu().item())


def beam_assign(instance: AssignmentInstance, beam_width: int = 2) -> Assignment:
    """Beam search over the greedy order, greedy kept as fallback
    (assignment.py:202-247), on device."""
    if beam_width < 1:
        raise AssignmentError(f"beam_width must be >= 1, got {beam_width}")
    if beam_width > _lib.MAX_BEAM:
        raise AssignmentError(f"beam_width must be <= {_lib.MAX_BEAM} on the device solver, "
                              f"got {beam_width}")
    C_, G_, _ = _run_policy(instance, 3, beam_width=beam_width)
    return Assignment(C=C_, G=G_)


def optimal_assign_with_stats(instance: AssignmentInstance,
                              max_activated: int = EXACT_SOLVER_LIMIT):
    """Exact minimum-makespan placement by branch and bound with the
    reference's bound, branch order and tie-break (assignment.py:268-346),
    on device.  Returns (assignment, makespan, explored nodes)."""
    n_act = len(instance.activated)
    if n_act > max_activated:
        raise AssignmentError(
            f"exact solver limited to {max_activated} activated experts, instance has "
            f"{n_act}; use greedy_assign instead")
    C_, G_, nodes = _run_policy(instance, 4, limit=max_activated)
    a = Assignment(C=C_, G=G_)
    if a == greedy_assign(instance):
        mk = makespan(instance, a)[2]
    else:                       # incumbent's lane totals accumulate in visit order
        order = instance.sorted_order()
        tc = tg = 0.0
        for e in order:
            if a.G[e]:
                tg += float(instance.gpu_times[e])
            else:
                tc += float(instance.cpu_times[e])
        mk = max(tc, tg)
    return a, float(mk), nodes


def optimal_assign(instance: AssignmentInstance, max_activated: int = EXACT_SOLVER_LIMIT):
    a, mk, _ = optimal_assign_with_stats(instance, max_activated)
    return a, mk


def static_threshold_assign(instance: AssignmentInstance,
                            threshold: float | None = None) -> Assignment:
    """GPU iff w >= threshold (default: median positive workload); capacity
    overflow to the CPU in descending-workload order (assignment.py:349-377)."""
    C_, G_, _ = _run_policy(instance, 5, threshold=threshold)
    return Assignment(C=C_, G=G_)
