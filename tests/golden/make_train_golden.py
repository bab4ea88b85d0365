"""Golden histories of config-driven training on the reference's CPU tiles.

Writes tests/golden/train/<name>.json -- the four experiments the reference
ships as proj/configs/*.json (ReRAM ExpStep MLP, Tiki-Taka, a conv net, a
PCM inference-family net), restated as dicts below -- and
tests/golden/train/<name>.csv, the epoch history of
integration/_ref/train_config_ref (the reference's parse_config /
build_network / train with its own tiles; needs /root/reference at build
time).  tests/test_gpu_cpp.py runs the same configs through
integration/_ref/train_config_b200 (every tile on the GPU) and compares.

    make -C integration && python tests/golden/make_train_golden.py
"""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "train")

BLOBS4 = {"kind": "blobs", "samples": 100, "features": 4, "classes": 2, "spread": 0.15}
IO7_9 = {"dac_bits": 7, "adc_bits": 9, "sigma_out": 0.06}

CONFIGS = {
    "train_reram": {
        "seed": 1234,
        "tile": {"family": "single", "device": {"preset": "reram_es"},
                 "forward_io": IO7_9, "backward_io": IO7_9, "update": {"bl": 31}},
        "network": {"layers": [{"type": "linear", "in": 4, "out": 2, "bias": "digital"}],
                    "loss": "mse"},
        "training": {"lr": 0.1, "epochs": 100, "batch_size": 10, "dataset": BLOBS4},
    },
    "tiki_taka": {
        "seed": 1234,
        "tile": {"family": "transfer",
                 "transfer": {"devices": [{"preset": "reram_sb", "dw_min_dtod": 0.1},
                                          {"preset": "reram_sb", "dw_min_std": 0.2}],
                              "units_in_mbatch": True, "transfer_every": 2,
                              "transfer_lr": 0.1, "columns_per_event": 1, "gamma": 1.0},
                 "forward_io": IO7_9, "backward_io": IO7_9},
        "network": {"layers": [{"type": "linear", "in": 4, "out": 2, "bias": "digital"}],
                    "loss": "mse"},
        "training": {"lr": 0.1, "epochs": 100, "batch_size": 10, "dataset": BLOBS4},
    },
    "conv_digits": {
        "seed": 1234,
        "tile": {"family": "single",
                 "device": {"kind": "constant_step", "dw_min": 0.001, "w_max": 1.0,
                            "w_min": -1.0},
                 "forward_io": {"dac_bits": 7, "adc_bits": 9, "sigma_out": 0.02}},
        "network": {"layers": [{"type": "conv2d", "in_channels": 1, "out_channels": 4,
                                "kernel": 3, "stride": 1, "padding": 0, "in_h": 8, "in_w": 8,
                                "activation": "relu"},
                               {"type": "linear", "in": 144, "out": 4, "bias": "digital"}],
                    "loss": "cross_entropy"},
        "training": {"lr": 0.05, "epochs": 20, "batch_size": 8,
                     "dataset": {"kind": "blobs", "samples": 64, "features": 64,
                                 "classes": 4, "spread": 0.2}},
    },
    "inference_pcm": {
        "seed": 1234,
        "tile": {"family": "inference",
                 "device": {"kind": "constant_step", "dw_min": 0.001, "w_max": 2.0,
                            "w_min": -2.0},
                 "forward_io": {"is_perfect": True}, "backward_io": {"is_perfect": True},
                 "inference": {"prog_noise_scale": 0.02, "c0": 0.26, "c1": 1.66, "c2": 0.33,
                               "read_noise_scale": 0.02, "nu_mean": 0.06, "nu_std": 0.3,
                               "t0": 1.0, "compensation_probes": 10}},
        "network": {"layers": [{"type": "linear", "in": 6, "out": 12, "bias": "digital",
                                "activation": "tanh"},
                               {"type": "linear", "in": 12, "out": 3, "bias": "digital"}],
                    "loss": "cross_entropy"},
        "training": {"lr": 0.1, "epochs": 40, "batch_size": 10,
                     "hw_aware": {"perfect_backward": True, "perfect_update": True,
                                  "weight_noise_sigma": 0.02},
                     "dataset": {"kind": "blobs", "samples": 300, "features": 6, "classes": 3,
                                 "spread": 0.25}},
    },
}


def main():
    os.makedirs(OUT, exist_ok=True)
    exe = os.path.join(ROOT, "integration", "_ref", "train_config_ref")
    for name, cfg in CONFIGS.items():
        path = os.path.join(OUT, name + ".json")
        with open(path, "w") as f:
            json.dump(cfg, f, indent=1)
            f.write("\n")
        r = subprocess.run([exe, path], capture_output=True, text=True, check=True)
        with open(os.path.join(OUT, name + ".csv"), "w") as f:
            f.write(r.stdout)
        print(name, r.stdout.splitlines()[-1])


if __name__ == "__main__":
    main()
