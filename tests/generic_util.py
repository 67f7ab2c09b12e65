"""Helpers for the generic-kernel tests: run a plan's KernelIRs on the
reference's own virtual SIMT device (oracle/_ref, vm::launch at
proj/src/vm.cpp:450-479) -- the semantics host/cudagen.cpp reproduces on the
GPU.  Test infrastructure only."""
import os
import re

import numpy as np

ATOMIC_GLOBAL = re.compile(r"atomic global (\w+)\[")
GENERIC_MF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "generic.mf")

# Scripts over tests/golden/generic.mf (user functions outside the algebra
# of the hand-written families).
USER_SCRIPTS = {
    "mul_add": ("subvector32 a, b, c, t, o;\ninput a, b, c;\nt = mul(a, b);\no = add(t, c);\n"
                "return o;\n", 1, 4096),
    "rscale_sgemv": ("TILE32x32 A, B;\nsubvector32 d, e, x, y;\ninput A, d, e, x;\n"
                     "B = rscale(A, d, e);\ny = sgemv(B, x);\nreturn B, y;\n", 96, 160),
}


def accumulated(kernel_text):
    """Buffers a kernel adds into with global atomics (the VM's contract:
    the caller zeroes them, proj/include/mapfuse/vm.hpp:91-93)."""
    return sorted(set(ATOMIC_GLOBAL.findall(kernel_text)))


def host_buffers(plan, values, rng=None):
    """Every buffer of the plan (intermediates too) as 2-D float32 arrays."""
    out = {}
    for b in plan.describe()["buffers"]:
        name, shape = b["name"], (b["rows"], b["cols"])
        if name in values and isinstance(values[name], np.ndarray):
            out[name] = np.ascontiguousarray(values[name], np.float32).reshape(shape).copy()
        elif b["role"] == "input" and rng is not None:
            out[name] = rng.uniform(-1, 1, shape).astype(np.float32)
        else:
            out[name] = np.zeros(shape, np.float32)
    return out


def vm_kernel(ref, plan, k, host, scalars):
    """Kernel k of the plan on the reference VM, in place; race-free asserted."""
    text = plan.kernel_text(k)
    for name in accumulated(text):
        host[name][...] = 0.0
    info = ref.vm_launch(text, host, scalars, poison=True, trace=True)
    assert info["hazards"] == 0, (plan.describe()["kernels"][k]["name"], info)
    return info


def vm_plan(ref, plan, host, scalars):
    for k in range(plan.num_kernels):
        vm_kernel(ref, plan, k, host, scalars)
    return host
