"""B200-native drop-in for the reference's `gsrecon` mini-BA surface
(config, scene, miniba). The LM work runs in paper_2506_05558_b200/libminiba.so."""
