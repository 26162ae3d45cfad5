"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NONE of the DMSGM arithmetic (no warp, mix, update or
classification).  It only draws frames, homographies, ground-truth object masks
and random model states.  See DESIGN.md §4 (input recipe).
"""
from .sequence import (CONFIGS, SeqConfig, Sequence, generate, generate_device, config, stream_rng,
                       camera_pose, homographies_for_stream, render_frame)
from .states import random_state, random_homography, blocks_of

__all__ = ["CONFIGS", "SeqConfig", "Sequence", "generate", "generate_device", "config", "stream_rng",
           "camera_pose", "homographies_for_stream", "render_frame",
           "random_state", "random_homography", "blocks_of"]
