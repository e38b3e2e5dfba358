"""Named workload presets C1–C5 (BASELINE.json `configs`).

Pure data: no arithmetic of the method lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

DAILY_DT = 1.0 / 252.0
MINUTE_DT = 1.0 / (252.0 * 390.0)


@dataclass(frozen=True)
class Workload:
    name: str
    n_stocks: int
    n_feat: int
    T_data: int
    dt: float
    n_envs: int          # per GPU
    T: int               # rollout length per call
    horizon: int         # episode length H
    n_hidden: int
    hidden: int
    n_agents: int        # per GPU
    h_max: int = 100
    C0: float = 1.0e6
    cost: float = 0.002
    reward_scale: float = 1.0
    gamma: float = 0.99
    lam: float = 0.95
    seed: int = 5188
    description: str = ""

    @property
    def obs_dim(self) -> int:
        return 1 + 2 * self.n_stocks + self.n_stocks * self.n_feat


PRESETS = {
    # configs[0]: oracle-scale
    "C1": Workload("C1", 30, 3, 2611, DAILY_DT, 16, 64, 64, 2, 128, 1, seed=5189,
                   description="Dow-30 daily synthetic prices, 16 envs, "
                               "T=64, actor MLP 2x128, single agent"),
    # configs[1]
    "C2": Workload("C2", 30, 3, 2611, DAILY_DT, 4096, 256, 1024, 2, 128, 1, seed=5190,
                   description="Dow-30 daily, 4096 envs per GPU, T=256, PPO rollout + GAE on 1xB200"),
    # configs[2]: the headline bench workload
    "C3": Workload("C3", 100, 3, 982_800, MINUTE_DT, 8192, 256, 8192, 3, 512, 1, seed=5191,
                   description="NASDAQ-100 minute-level synthetic (10y, 8192-step horizon chunks), "
                               "8192 envs per GPU, actor MLP 3x512"),
    # configs[3]
    "C4": Workload("C4", 100, 3, 982_800, MINUTE_DT, 8192, 256, 8192, 3, 512, 8, seed=5192,
                   description="Generational evolution: 8 agents per GPU; fitness all-gather + "
                               "top-k elite broadcast each generation"),
    # configs[4]
    "C5": Workload("C5", 100, 3, 982_800, MINUTE_DT, 65536, 1024, 8192, 3, 512, 1, seed=5193,
                   description="Ensemble stress: NASDAQ-100 minute, 65536 envs per GPU, T=1024, bf16 actor"),
}


def preset(name: str, **overrides) -> Workload:
    return replace(PRESETS[name], **overrides)
