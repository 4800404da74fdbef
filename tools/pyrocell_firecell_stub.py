"""The maintainer-side binding INTEGRATION.md shows: what pyrocell would add
(as ``pyrocell/_firecell.py``) to route its step loop through libfirecell.so
with ctypes.  Kept as a module so the tests execute exactly the text the
documentation shows (tests/test_abi_host.py checks its calls against the
header's arities; tests/test_gpu_parity.py runs it against FireBatch.run)."""
import ctypes as C

import torch

from paper_2502_18738_b200 import _lib as L  # struct layouts + argtypes (include/firecell.h)

lib = L.lib()  # raises RuntimeError if libfirecell.so is missing: no CPU fallback


def run_device(batch, land_dev, nsteps, attach_flags=None, window=8):
    """pyrocell/kernel.py:504-524 (the run_simulation step loop) as one fc_run
    call: `window` steps fused per launch, keyed SplitMix draws (rng.py:55-75),
    activity skipping on, no wind schedule, no shard."""
    att = None if attach_flags is None else (C.c_uint8 * nsteps)(*attach_flags)
    phase = C.c_int32(batch.q)                       # launches since reset (in/out)
    rc = lib.fc_run(C.byref(batch.grid), C.byref(land_dev.struct()), C.byref(batch.struct()),
                    batch.params.data_ptr(), batch.seeds.data_ptr(),
                    L.RNG_SPLITMIX,                  # rng_mode
                    None,                            # draws (FC_RNG_INJECT only)
                    batch.t, nsteps,                 # t0, nsteps
                    att,                             # host_attach
                    1,                               # skip_inactive
                    window,                          # steps per launch
                    None,                            # wind_schedule
                    None,                            # shard
                    C.byref(phase),                  # host_phase
                    torch.cuda.current_stream().cuda_stream)
    L.check(rc, "fc_run")                            # FC_EINVAL -> ValueError
    batch.t += nsteps
    batch.q = phase.value


def contract_device(batch, dl_dacc):
    """pyrocell/tape.py:118-148 (backward_params) for one member: sum over the
    run's ignitions of dL/dacc * J, fp64, on the device."""
    g = torch.as_tensor(dl_dacc, dtype=torch.float64, device=batch.device).contiguous()
    out = torch.empty((batch.m, 4), dtype=torch.float64, device=batch.device)
    rc = lib.fc_contract(C.byref(batch.grid), C.byref(batch.struct()), g.data_ptr(),
                         0,                          # g is fp64
                         out.data_ptr(), batch.workspace.data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
    L.check(rc, "fc_contract")
    return out
