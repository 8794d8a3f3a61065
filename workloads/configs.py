"""The five BASELINE.json configurations (SURVEY §8(d) input recipe).

Each config names the topology, the frame geometry, chunk length L, chunks per
step B, the synthetic-video recipe and the threshold policy.  cfg ids are
1-based like SURVEY (cfg1 = BASELINE.json configs[0]).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

from . import models

SEED_BASE = 2410207900


@dataclass
class Config:
    cid: int
    name: str
    model: str
    h: int
    w: int
    c: int
    L: int
    chunks_per_step: int
    steps: int
    video: dict = field(default_factory=dict)
    policy: str = "fixed"          # fixed | bst | ibst
    theta_fixed: float = 0.05
    T: float = 0.9
    eps: float = 0.05
    cycle: int = 8
    note: str = ""

    def build_net(self, weight_seed=None, calibrated=True):
        """Topology + seeded weights; with ``calibrated`` (and the default
        seed) the committed per-channel BatchNorm fold of reading R30
        (workloads/calib/cfg<N>.npz, written once by
        scripts/calibrate_weights.py) is applied when it exists."""
        builders = {"toy": models.toy_encoder, "crnn": models.crnn_vgg7,
                    "resnet18": models.resnet18, "effb0": models.efficientnet_b0,
                    "resnet152": models.resnet152}
        for v in ("b4", "b5", "b6"):
            builders["eff" + v] = (lambda vv: lambda h, w: models.efficientnet(h, w, vv))(v)
        net = builders[self.model](self.h, self.w)
        models.init_weights(net, SEED_BASE + 1000 * self.cid + 999 if weight_seed is None else weight_seed)
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "calib", f"cfg{self.cid}.npz")
        if calibrated and weight_seed is None and os.path.exists(path):
            models.apply_fold(net, path)
        return net

    def video_seed(self, chunk):
        return SEED_BASE + 1000 * self.cid + chunk


CONFIGS = {
    1: Config(1, "toy", "toy", 64, 64, 3, L=8, chunks_per_step=1, steps=1,
              video=dict(n_objects=3, size=(8, 16), speed=(1, 1), frames_per_px=2,
                         noise_q=0.05, noise_amp=1),
              policy="fixed", theta_fixed=0.05,
              note="toy encoder, one 8-frame chunk of 64x64x3 slow-motion video, threshold 0.05"),
    2: Config(2, "crnn", "crnn", 32, 128, 1, L=32, chunks_per_step=64, steps=4,
              video=dict(text=True, n_objects=0, frames_per_px=2, noise_q=0.05, noise_amp=1),
              policy="fixed", theta_fixed=0.05,
              note="CRNN VGG-7 conv encoder, 32-frame chunks of 32x128 grayscale synthetic text video"),
    3: Config(3, "effb0_512", "effb0", 512, 512, 3, L=16, chunks_per_step=8, steps=16,
              video=dict(n_objects=12, size=(16, 96), speed=(1, 3), noise_q=0.10, noise_amp=2),
              policy="ibst", T=0.9, eps=0.05, cycle=8,
              note="EfficientNet-B0 backbone @512x512, 16-frame chunks, online threshold adjustment"),
    4: Config(4, "resnet18_720p", "resnet18", 720, 1280, 3, L=32, chunks_per_step=8, steps=1,
              video=dict(n_objects=10, size=(96, 320), speed=(1, 4), noise_q=0.10, noise_amp=2),
              policy="bst", T=0.9, eps=0.02,
              note="ResNet-18 @720p, 32-frame chunks, sparsity sweep"),
    5: Config(5, "effdet_d0_1080p", "effb0", 1080, 1920, 3, L=16, chunks_per_step=8, steps=8,
              video=dict(n_objects=12, size=(32, 192), speed=(1, 3), noise_q=0.10, noise_amp=2),
              policy="ibst", T=0.9, eps=0.05, cycle=8,
              note="EfficientDet-D0 backbone @1080p, 64 chunks, chunk-sharded over GPUs"),
    # SURVEY §8(f) N3 (not a BASELINE.json config): the paper's own CRNN
    # backbone, ResNet-152 at 320x320, chunks of 28 frames, 3 chunks per step
    6: Config(6, "resnet152_320", "resnet152", 320, 320, 3, L=28, chunks_per_step=3, steps=4,
              video=dict(n_objects=6, size=(32, 96), speed=(1, 3), noise_q=0.10, noise_amp=2),
              policy="ibst", T=0.9, eps=0.05, cycle=8,
              note="ResNet-152 CRNN backbone @320x320, 28-frame chunks, batch 3 (N3)"),
    # the Table 1 detectors' backbones,
    # EfficientDet-d4 / d5 / d6 = EfficientNet-B4 @1024 / B5 @1280 / B6 @1280,
    # on static-camera street video like cfg5 (MOT16), 16-frame chunks
    7: Config(7, "effdet_d4_1024", "effb4", 1024, 1024, 3, L=16, chunks_per_step=2, steps=4,
              video=dict(n_objects=10, size=(32, 160), speed=(1, 3), noise_q=0.10, noise_amp=2),
              policy="ibst", T=0.9, eps=0.05, cycle=8,
              note="EfficientDet-d4 backbone (EfficientNet-B4) @1024x1024, 16-frame chunks (N3)"),
    8: Config(8, "effdet_d5_1280", "effb5", 1280, 1280, 3, L=16, chunks_per_step=2, steps=4,
              video=dict(n_objects=12, size=(32, 192), speed=(1, 3), noise_q=0.10, noise_amp=2),
              policy="ibst", T=0.9, eps=0.05, cycle=8,
              note="EfficientDet-d5 backbone (EfficientNet-B5) @1280x1280, 16-frame chunks (N3)"),
    9: Config(9, "effdet_d6_1280", "effb6", 1280, 1280, 3, L=16, chunks_per_step=2, steps=4,
              video=dict(n_objects=12, size=(32, 192), speed=(1, 3), noise_q=0.10, noise_amp=2),
              policy="ibst", T=0.9, eps=0.05, cycle=8,
              note="EfficientDet-d6 backbone (EfficientNet-B6) @1280x1280, 16-frame chunks (N3)"),
    # the paper's CRNN experiments at its other two resolutions
    10: Config(10, "resnet152_224", "resnet152", 224, 224, 3, L=28, chunks_per_step=3, steps=4,
               video=dict(n_objects=5, size=(24, 72), speed=(1, 3), noise_q=0.10, noise_amp=2),
               policy="ibst", T=0.9, eps=0.05, cycle=8,
               note="ResNet-152 CRNN backbone @224x224, 28-frame chunks, batch 3 (N3)"),
    11: Config(11, "resnet152_420", "resnet152", 420, 420, 3, L=28, chunks_per_step=3, steps=4,
               video=dict(n_objects=8, size=(40, 128), speed=(1, 3), noise_q=0.10, noise_amp=2),
               policy="ibst", T=0.9, eps=0.05, cycle=8,
               note="ResNet-152 CRNN backbone @420x420, 28-frame chunks, batch 3 (N3)"),
}


def get_config(cid: int) -> Config:
    return CONFIGS[cid]
