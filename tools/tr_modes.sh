#!/bin/bash
# hooks modes A/B (train_overhead.py) on the three bench models
timeout 900 python tools/train_overhead.py resnet50 256 hooks_codec_bf1,hooks_codec,hooks_codec_bf1,hooks_codec 2>&1 | grep -v Warn | grep "b256\|per-it"
timeout 700 python tools/train_overhead.py alexnet 256 plain,hooks_codec_bf1,hooks_codec 2>&1 | grep -v Warn | grep "b256"
timeout 700 python tools/train_overhead.py vgg16 128 hooks_codec_bf1,hooks_codec 2>&1 | grep -v Warn | grep "b128"
