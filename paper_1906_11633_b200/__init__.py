"""B200-native batched domain-randomization pipeline behind the C-ABI libdr.so.

``dr``      -- thin ctypes binding, same names as include/dr.h
``DRContext`` -- convenience owner of one context: torch-allocated outputs and stats buffer
"""
from . import dr  # noqa: F401


class DRContext:
    """One libdr context on the current CUDA device (one per process).

    Allocates the output tensors and a caller-owned [4][32] fp64 stats ring (so NCCL can
    all-reduce it), and passes torch's current stream to the library.  Marshalling only."""

    def __init__(self, preset: dict, n_env: int, seed: int, env_offset: int = 0, n_env_global: int = 0,
                 stream=None, workspace: bool = False):
        import torch
        self.n = int(n_env)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        ws = None
        params = dr.params_from_preset(preset, env_offset=env_offset, n_env_global=n_env_global,
                                       stream=self.stream.cuda_stream)
        if workspace:
            nbytes = dr.dr_workspace_bytes(params, self.n)
            ws = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
            off = (-ws.data_ptr()) % 256
            ws = ws[off:off + nbytes]
            params = dr.params_from_preset(preset, env_offset=env_offset, n_env_global=n_env_global,
                                           stream=self.stream.cuda_stream, workspace=ws)
        self._ws = ws
        self._env_offset, self._n_env_global = env_offset, n_env_global
        self.preset = preset
        dr.dr_init(params, self.n, seed)
        self._open = True
        dev = "cuda"
        self.stats = torch.zeros(dr.N_STAT_SLOTS, dr.N_STATS, dtype=torch.float64, device=dev)
        dr.dr_set_stats_buffer(self.stats)
        self.out_actions = torch.empty(self.n, dr.N_ACT, device=dev)
        self.out_obs = torch.empty(self.n, dr.OBS_OUT, device=dev)
        self.out_dt = torch.empty(self.n, dr.N_SUB, device=dev)
        self.out_force = torch.empty(self.n, 3, device=dev)
        self.substeps = bool(preset["layer_mask"] & dr.SUBSTEP_BACKLASH)
        self.out_actions_sub = torch.empty(self.n, dr.N_SUB, dr.N_ACT, device=dev) if self.substeps else None

    def step(self, actions, raw_obs, outs=None):
        o = outs or (self.out_actions, self.out_obs, self.out_dt, self.out_force)
        if self.substeps:   # DR_SUBSTEP_BACKLASH: one gated action per substep as well
            dr.dr_step_substeps(actions, raw_obs, o[0], self.out_actions_sub, *o[1:])
        else:
            dr.dr_step(actions, raw_obs, *o)
        return o

    def update_params(self, preset: dict, env_offset: int = None, n_env_global: int = None):
        """dr_update_params with a preset dict (same shape/layers/shard as at init)."""
        params = dr.params_from_preset(preset, env_offset=self._env_offset if env_offset is None else env_offset,
                                       n_env_global=self._n_env_global if n_env_global is None else n_env_global,
                                       stream=self.stream.cuda_stream)
        dr.dr_update_params(params)
        self.preset = preset

    def reset(self, mask=None):
        dr.dr_reset(mask, self.n if mask is not None else None)

    def last_stats(self):
        """fp64 stats of the most recent step (synchronises; the slot comes from the device step
        counter, which CUDA-graph replays advance too)."""
        t = dr.dr_step_index_sync()
        return self.stats[(t - 1) % dr.N_STAT_SLOTS].cpu().numpy()

    def export(self, lo: int = 0, hi: int = 0) -> dict:
        return dr.states_to_numpy(dr.dr_state_export(lo, hi))

    def phys(self, lo: int = 0, hi: int = 0):
        return dr.dr_phys_export(lo, hi)

    def close(self):
        if self._open:
            dr.dr_finalize()
            self._open = False

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
