"""B200-native (sm_100a) reduced-objective hot path of arXiv 2409.03807.

Public API (mirrors the reference `lipsub` names): see paper_2409_03807_b200.lipsub.
All compute runs in the in-tree CUDA library _lib/liblipsub_b200.so through the C ABI
declared in include/lipsub_b200.h; importing works without a GPU, calling does not.
"""
from .lipsub import *  # noqa: F401,F403
from .lipsub import (Activation, ExitCode, ExitReport, FrameInput, Layer, Mesh, ReducedObjective,  # noqa: F401
                     ReducedSystem, SimState, SolverConfig, SubspaceModel, build_mesh, dof_pack, dof_unpack,
                     gravity_force, lame_from_young, lbfgs_minimize, lipschitz_loss, make_bar_decoder,
                     lipschitz_loss_grad, make_bar_mesh, reduced_step, rest_state)
from ._capi import LibraryMissing, LsbError, lib  # noqa: F401
from .checkpoint import load_checkpoint, save_checkpoint  # noqa: F401
from .scenario import (Scenario, frame_at, load_node_ele, load_scenario, make_bar_3d, pin_positions_at,  # noqa: F401
                       replay_interactions, sample_interaction, scenario_from_json)
